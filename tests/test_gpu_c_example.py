"""The C ABI from plain C (examples/quantize.c, built by __graft_entry__.build()): init, solve,
labels with palette, free - no Python or torch in the process. Four noisy quadrants must come out
as four clusters whose palette entries are the quadrant colours."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("H,W", [(96, 128), (61, 77)])
def test_c_example_quantizes(H, W):
    import __graft_entry__ as g
    exe = g.build_examples()
    r = subprocess.run([exe, str(H), str(W)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.split()[0] == "ok" and r.stdout.split()[4] == "4", r.stdout
