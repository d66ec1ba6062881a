"""Share of device time per kernel in an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).

    python profiles/summarize_launches.py profiles/r1_launches_c2_v2.csv
"""
import csv
import sys

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
         "s": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = {}, {}
    for r in rows[start + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0]
        ms = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        tot[name] = tot.get(name, 0.0) + ms
        cnt[name] = cnt.get(name, 0) + 1
    total = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {total:.3f} ms of device time")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
        print(f"{v:10.3f} ms  {100 * v / total:5.1f} %  x{cnt[k]:<4d} {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
