"""Freeze the algorithmic bytes per ray*bounce of each config:

    B_rb = 64*n_int + 48*n_leaf + 48 + 4 + 128/b_bar

n_int / n_leaf are counted by the oracle (oracle/roomray_oracle.c, the
reference traversal order of accel_tree.cpp:141-179: pops surviving the
prune) over build_tree's tree on a strided subset of each config's lattice;
b_bar = ray*bounces per ray.  Counted on the reference's algorithm, never on
the GPU kernel, so kernel changes cannot move the denominator.  Writes
profiles/brb_frozen.json (existing entries are kept unless --force).

    python profiles/freeze_brb.py [c1 c2 c3 c5] [--force]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1811_05784_b200 import scenes  # noqa: E402

STRIDES = {"c1": 1, "c2": 97, "c3": 5, "c5": 4001}


def freeze(name, stride):
    s = scenes.CONFIGS[name]()
    port = oracle.Port()
    sc = port.scene(oracle.Mesh(s.vertices, s.faces, s.absorption))
    rc = [c for c, _ in s.receivers]
    rr = [r for _, r in s.receivers]
    _, st = sc.trace(s.source, s.ray_count, rc, rr, s.max_iterations, s.max_range, os.cpu_count() or 1, 0, stride,
                     0)
    rays = (s.ray_count + stride - 1) // stride
    n_int = st.sum_n_int / st.ray_bounces
    n_leaf = st.sum_n_leaf / st.ray_bounces
    b_bar = st.ray_bounces / rays
    return {"B_rb": 64 * n_int + 48 * n_leaf + 48 + 4 + 128 / b_bar, "n_int": n_int, "n_leaf": n_leaf,
            "b_bar": b_bar,
            "counted_on": f"oracle/roomray_oracle.c nearest_hit counters (accel_tree.cpp:141-179 order, pops "
                          f"surviving the prune) over build_tree's tree; {rays} lattice rays (k = 0 mod {stride}), "
                          f"{st.ray_bounces} ray*bounces",
            "formula": "64*n_int + 48*n_leaf + 48 + 4 + 128/b_bar (SURVEY.md 8(d))",
            "ncu_dram_bytes_per_launch": None}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    force = "--force" in sys.argv
    path = os.path.join(ROOT, "profiles", "brb_frozen.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    oracle.build(ref=False)
    for name in args or list(STRIDES):
        if name in data and not force:
            continue
        data[name] = freeze(name, STRIDES[name])
        print(name, json.dumps(data[name]))
    json.dump(data, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
