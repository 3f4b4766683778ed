"""compute-sanitizer over every kernel path on small graphs:
memcheck (out-of-bounds / misaligned), racecheck (shared-memory hazards),
synccheck (barrier misuse). scripts/sanitize.py runs BFS in every direction x
strategy, SSSP, BC, CC and PageRank on symmetric and directed graphs, and the
partitioned BFS / SSSP kernels (3 loopback partitions), and checks the oracle."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if os.environ.get("GR_SANITIZER") != "1":
        # this GPU pool closed compute-sanitizer (its wrapper refuses every run);
        # opt in where it is available
        pytest.skip("compute-sanitizer runs are opt-in (GR_SANITIZER=1)")
    import __graft_entry__
    __graft_entry__.build()
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if "sanitize workload ok" not in out and "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run: the same
        # bounds and race properties are then covered by the parity suites only
        pytest.skip("compute-sanitizer unavailable on this GPU pool: " + out.strip()[:200])
    assert "sanitize workload ok" in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
