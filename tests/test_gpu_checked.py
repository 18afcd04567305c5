"""The sanitizer substitute (compute-sanitizer is closed on this GPU pool): tools/sanitize_small.py under the
checked library build (mbarrier watchdogs, device bounds checks), poisoned allocations (NaN: reads before
writes) and canary tails (out-of-bounds writes), plus bitwise run-to-run reproducibility of the parameters, over
every step-kernel variant. Runs in a subprocess so that the checked library is the one loaded."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lib", ["liblcae_checked.so", "liblcae.so"])
def test_sanitizer_substitute(lib):
    path = os.path.join(ROOT, "paper_1502_03409_b200", lib)
    assert os.path.exists(path), f"{lib} not built (make -C paper_1502_03409_b200/csrc)"
    env = dict(os.environ, LCAE_LIB=path, LCAE_DEV_POISON="1", LCAE_DEV_CANARY="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_small.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "sanitize run ok" in r.stdout
