"""CPU: bench.py's multi-GPU launcher.  `--gpus 2 --dry-run` re-launches
itself under torch.distributed.run as 2 gloo ranks, each derives its
block-cyclic shard of the C5 lattice the way run_trace does, and rank 0
prints n_gpus 2 with the shards summing to the whole lattice; a torchrun
world size that disagrees with --gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _last_json(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_dry_run_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--dry-run"], capture_output=True, text=True,
                       timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    j = _last_json(p.stdout)
    assert j["n_gpus"] == 2 and j["dry_run"] and j["scaling"] == "strong"
    assert j["rays_total"] == j["lattice"] == 8_000_000
    assert j["max_over_ranks"] == 2.0  # the MAX reduction saw both ranks
    assert 0 < j["rays_rank0"] < 8_000_000


def test_world_size_mismatch_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, BENCH, "--gpus", "4", "--dry-run"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr


def test_roofline_counters_from_committed_ncu_exports():
    """bench.py's roofline reads the committed raw ncu exports of the trace
    kernel (profiles/ncu_trace_<cfg>.csv): DRAM read + write bytes, L2 bytes,
    duration, and the issue-slot counters, per launch."""
    sys.path.insert(0, ROOT)
    import bench
    for cfg in ("c5", "c3", "c2"):
        c = bench.ncu_trace_counters(cfg)
        assert c is not None and c["launches"] == 1, cfg
        assert c["dram_bytes"] == c["dram_read"] + c["dram_write"] > 0
        assert c["l2_bytes"] > c["dram_bytes"]
        assert 0.1 < c["ncu_ms"] < 5000.0
        assert 0.0 < c["issue_active_pct"] <= 100.0 and 1.0 <= c["threads_per_inst"] <= 32.0
    c5 = bench.ncu_trace_counters("c5")
    assert 300 < c5["dram_bytes"] / 799_998_849 < 2000  # bytes per C5 ray*bounce
