"""CPU: the C-ABI library and host logic (no GPU calls).

* libroomray_b200.so loads and exports every function include/roomray_b200.h
  declares, and the ctypes signature table covers them all;
* scene generators are deterministic and have the BASELINE.json sizes;
* the device emission's sin/cos (rr_sincos.cuh, compiled for the host here)
  is bit-identical to the installed glibc sincos() -- the call the
  reference's fibonacci_directions makes -- on every lattice azimuth of every
  config and on random arguments in each branch; its correctly rounded
  fallback (beyond 1.05e8 rad) is checked against decimal sin.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1811_05784_b200 import _lib, scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "roomray_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rr_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(syms) <= bound, set(syms) - bound
    assert lib.rr_version  # noqa


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_string():
    lib = _lib.load()
    assert b"sm_100a" in lib.rr_version()


def test_host_alloc_argument_errors():
    # no device needed: size 0 returns NULL, a negative size is RR_INVALID_ARGUMENT, free(NULL) is a no-op
    lib = _lib.load()
    p = ctypes.c_void_p(1)
    assert lib.rr_host_alloc(0, ctypes.byref(p)) == 0 and p.value is None
    assert lib.rr_host_alloc(-8, ctypes.byref(p)) == 1
    assert b"bytes" in lib.rr_last_error()
    assert lib.rr_host_free(None) == 0


def test_splitmix_golden_values():
    # splitmix64 reference outputs for seed 0 (first three)
    z = scenes.splitmix64(0, 3)
    assert [hex(int(x)) for x in z] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]


def test_config_sizes_and_determinism():
    c1, c2 = scenes.config1(), scenes.config2()
    assert c1.n_faces == 1200 and c2.n_faces == 100_000
    assert np.array_equal(scenes.config2().absorption, c2.absorption)
    assert (c2.absorption >= 0.02).all() and (c2.absorption < 0.4).all()
    lo, hi = c2.vertices.min(0), c2.vertices.max(0)
    np.testing.assert_array_equal(lo, [0, 0, 0])
    np.testing.assert_array_equal(hi, [8, 6, 3])
    # closed box: every edge is shared by exactly two triangles
    f = c1.faces[:, :3]
    key = {tuple(np.round(c1.vertices[i], 9)) for i in f.reshape(-1)}
    assert len(key) == len({tuple(x) for x in np.round(c1.vertices, 9)})


def test_block_cyclic_partition_covers_each_ray_once():
    """Host side of the multi-GPU sharding (rr_trace_config.block): blocks of
    B rays round-robin over ranks; the union is the lattice, no overlap."""
    N, B = 100_003, 4096
    seen = np.zeros(N, int)
    for world in (1, 2, 4, 8):
        seen[:] = 0
        for rank in range(world):
            nblk = (N + B - 1) // B
            for blk in range(rank, nblk, world):
                seen[blk * B:min(N, (blk + 1) * B)] += 1
        assert (seen == 1).all()


@pytest.fixture(scope="module")
def sincos_check():
    exe = os.path.join(ROOT, "build", "sincos_check")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-I",
                    os.path.join(ROOT, "paper_1811_05784_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "sincos_check.cpp"), "-o", exe], check=True)
    return exe


def _sincos_run(exe, *args):
    out = subprocess.run([exe, *map(str, args)], capture_output=True, text=True).stdout
    m = re.search(r"mismatches (\d+) of (\d+) fallback (\d+)", out)
    assert m, out
    return int(m.group(1)), int(m.group(2)), int(m.group(3)), out


def test_emission_sincos_bit_identical_to_glibc_on_every_lattice(sincos_check):
    """Every azimuth of C1 (10^4 rays), C2/C3 (10^6) and C5 (8*10^6)."""
    bad, n, fb, out = _sincos_run(sincos_check, "lattice", 10_000, 1_000_000, 8_000_000)
    assert n == 9_010_000 and fb == 0
    assert bad == 0, out


def test_emission_sincos_bit_identical_to_glibc_random(sincos_check):
    """Random arguments in every branch of glibc's routine (tiny, Taylor,
    table, pi/2 - |x|, Cody-Waite up to 1.05e8 rad), both signs."""
    bad, n, fb, out = _sincos_run(sincos_check, "random", 4_000_000, 11)
    assert n > 3_900_000 and fb > 0
    assert bad == 0, out


def test_emission_sincos_correctly_rounded():
    """Spot-check rr::sincos_cr (the fallback beyond 1.05e8 rad) against
    60-digit decimal sin/cos on azimuths where glibc is not correctly
    rounded."""
    from decimal import Decimal, getcontext
    getcontext().prec = 60
    exe_src = os.path.join(ROOT, "tests", "native", "sincos_check.cpp")
    assert os.path.exists(exe_src)

    def dpi():
        def atan_inv(x):
            x = Decimal(x)
            s, t, n, x2, sg = Decimal(0), 1 / x, 1, x * x, 1
            while True:
                term = t / n
                if term < Decimal(10) ** -58:
                    return s
                s += sg * term
                t /= x2
                n += 2
                sg = -sg
        return 16 * atan_inv(5) - 4 * atan_inv(239)

    pi = dpi()

    def dsin(x):
        x = Decimal(x)
        k = (x / (2 * pi)).to_integral_value()
        r = x - k * 2 * pi
        s, t, n = Decimal(0), r, 1
        while abs(t) > Decimal(10) ** -58:
            s += t
            t = -t * r * r / ((n + 1) * (n + 2))
            n += 2
        return s

    golden = (1 + 5 ** 0.5) / 2
    step = 2 * np.pi * (1 - 1 / golden)
    for k, expect in [(232, -0.66654885887170978), (679, 0.79045668616243747), (899, 0.64971501957170041)]:
        phi = step * k
        assert float(dsin(phi)) == expect
