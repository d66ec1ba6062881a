"""Host side of the artifact writers (include/roomray_b200_artifacts.hpp):
the JSON number text must equal nlohmann::json's (the reference's writer,
pipeline.cpp via json.hpp) bit pattern for bit pattern, so equal values give
byte-identical files.  CPU only; needs the nlohmann header shipped in the
image (the cudnn-frontend copy, 3.11.3)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


@pytest.mark.skipif(not os.path.exists(os.path.join(JSON_DIR, "json.hpp")), reason="nlohmann json.hpp not in image")
def test_json_numbers_match_nlohmann(tmp_path):
    exe = str(tmp_path / "json_number_check")
    lib = os.path.join(ROOT, "paper_1811_05784_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-I", JSON_DIR,
                    os.path.join(ROOT, "tests", "native", "json_number_check.cpp"), "-L", lib, "-lroomray_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    r = subprocess.run([exe, "1000000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout


def test_io_round_trips(tmp_path):
    """tests/test_io.cpp restated on the facade's host IO: WAV float32 round
    trip, non-WAV / missing files fail cleanly, band-trains CSV round trip
    bit for bit, a bad band index names its line."""
    exe = str(tmp_path / "io_roundtrip")
    lib = os.path.join(ROOT, "paper_1811_05784_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "io_roundtrip.cpp"), "-L", lib, "-lroomray_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    out = tmp_path / "io"
    out.mkdir()
    r = subprocess.run([exe, str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "io ok" in r.stdout, r.stdout + r.stderr
