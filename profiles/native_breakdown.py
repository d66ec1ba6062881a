"""Stage breakdown of the C++ facade's run_trace_pipeline (profiles/native_breakdown.cpp)
on a bench config: device work vs device->host copies vs host-side struct building.

    python profiles/native_breakdown.py [c5] [steps] [warmup]

RR_BREAKDOWN_INCLUDE=<dir> compiles against another copy of the façade headers (A/B).
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    warmup = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    lib_dir = os.path.join(ROOT, "paper_1811_05784_b200")
    inc = os.environ.get("RR_BREAKDOWN_INCLUDE", os.path.join(ROOT, "include"))
    exe = os.path.join(ROOT, "build", "native_breakdown_" + str(abs(hash(inc)) % 10**6))
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", inc,
                    os.path.join(ROOT, "profiles", "native_breakdown.cpp"), "-L", lib_dir, "-lroomray_b200",
                    "-Wl,-rpath," + lib_dir, "-o", exe], check=True)
    scene = bench.load_scene(cfg)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "scene.bin")
        bench.write_scene_bin(scene, path)
        out = subprocess.run([exe, path, str(steps), str(warmup)], capture_output=True, text=True, check=True)
    print(cfg, "ms per step:", out.stdout.strip())


if __name__ == "__main__":
    main()
