"""SASS opcode mix of one kernel in an ncu report (SourceCounters), overall
and per source line for one opcode:
    python profiles/ncu_opmix.py <report.ncu-rep> [OPCODE [top]]"""
import collections
import csv
import io
import re
import subprocess
import sys


def page(rep, what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", f"--print-source={what}"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    # address -> (file, line) from the interleaved page
    where, cur_file, cur_line = {}, None, None
    for r in page(rep, "cuda,sass"):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].rsplit("/", 1)[-1]
        elif r[0].isdigit():
            cur_line = (cur_file, int(r[0]), r[1].strip()[:90])
        elif r[0] == "" and len(r) > 2 and r[2].startswith("0x"):
            where[r[2]] = cur_line
    rows = page(rep, "sass")
    h = rows[1]
    ie, te, src = h.index("Instructions Executed"), h.index("Thread Instructions Executed"), h.index("Source")
    ops, thr, per_line = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= ie or not r[ie].isdigit():
            continue
        s = re.sub(r"^@!?U?P\w+\s+", "", r[src].strip())
        op = (s.split() or ["?"])[0].split(".")[0]
        n = int(r[ie])
        ops[op] += n
        thr[op] += int(r[te])
        if want and op == want:
            per_line[where.get(r[0])] += n
    tot = sum(ops.values())
    if not want:
        for op, n in ops.most_common(top):
            print(f"{op:10s} {100 * n / tot:6.2f}%  threads/inst {thr[op] / max(n, 1):5.1f}")
        return
    for ln, n in per_line.most_common(top):
        print(f"{100 * n / tot:6.2f}% of all  {ln}")


if __name__ == "__main__":
    main()
