"""Per-source-line instruction / stall shares of one kernel in an ncu report:
python profiles/ncu_hot.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                         text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            ie, te = int(d["Instructions Executed"]), int(d["Thread Instructions Executed"])
            smp = int(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        rows.append((ie, te, smp, cur.split("/")[-1], int(r[0]), r[1].strip()[:90]))
    ti = sum(r[0] for r in rows) or 1
    ts = sum(r[2] for r in rows) or 1
    rows.sort(reverse=True)
    for ie, te, smp, f, ln, src in rows[:top]:
        print(f"{ie / ti * 100:5.1f}% inst {smp / ts * 100:5.1f}% stall-samples thr/inst {te / max(ie, 1):5.1f}  "
              f"{f}:{ln}  {src}")


if __name__ == "__main__":
    main()
