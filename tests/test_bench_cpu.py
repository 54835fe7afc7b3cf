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
