"""CPU checks of the bench harness: it imports without a GPU, accepts every config the
docs name, and the reference arm's bounded sample is sized for a few minutes."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_modules_import():
    sys.path.insert(0, ROOT)
    import bench  # noqa: F401
    import bench_extra

    assert hasattr(bench_extra, "run_extra") and hasattr(bench_extra, "_e2e")


def test_bench_accepts_every_config():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         cwd=ROOT, timeout=120)
    assert out.returncode == 0, out.stderr
    for c in ("C1", "C2", "C3", "C4", "C5", "N1", "N2", "N3", "N4"):
        assert c in out.stdout, c
    assert "--impl" in out.stdout and "--gpus" in out.stdout


def test_bench_gpus_flag_starts_that_many_ranks():
    """`bench.py --gpus 2` outside torchrun starts two ranks (gloo here, no GPU)."""
    import json

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--spawn-check"],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["world"] == 2 and sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2


def test_bench_refuses_mismatched_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                         text=True, cwd=ROOT, timeout=300, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_strong_scaling_partition_of_bench_configs():
    """C2/C5 at N=1,2,4,8: one global array, chunk starts aligned to 256, every rank
    but the last holds at least the largest window's halo."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_cs_0610046_b200 import shard

    for cfg in ("C2", "C5"):
        n, wmax = bench.CONFIGS[cfg]["n"], max(bench.CONFIGS[cfg]["windows"])
        for P in (1, 2, 4, 8):
            b = shard.split_even(n, P)
            assert b[0][0] == 0 and b[-1][1] == n and all(s % 256 == 0 for s, _ in b)
            assert all(e - s >= wmax - 1 for s, e in b)
