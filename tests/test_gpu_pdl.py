"""Programmatic dependent launch (PDL) does not change results: the update
chain with PDL (kernels overlapping their predecessors' tails) is bit-identical
to the fully serialised chain (DASH_NO_PDL=1) and across repeated runs, on a
large-shaped stream (20k small slices + 300 big slices per update)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _digest(no_pdl: bool, *args, **switches) -> str:
    env = dict(os.environ)
    for k in ("DASH_NO_PDL", "DASH_NO_SIDE_PLAN"):
        env.pop(k, None)
    if no_pdl:
        env["DASH_NO_PDL"] = "1"
    env.update(switches)
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "pdl_check.py"), *args], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


def test_pdl_chain_is_bit_identical_to_serialised_chain():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _digest(False)
    b = _digest(False)
    c = _digest(True)
    assert a == b == c, (a, b, c)


def test_side_stream_plan_is_bit_identical_to_in_stream_plan():
    """The device plan of update t+1 running on the staging side stream while update t executes
    (double-buffered plan sets, event hand-off) changes nothing: updates issued back to back
    without host syncs give the same bytes as with DASH_NO_SIDE_PLAN=1, as with per-update
    syncs, and as with PDL off."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _digest(False, "async")
    b = _digest(False, "async", DASH_NO_SIDE_PLAN="1")
    c = _digest(False)
    d = _digest(True, "async")
    assert a == b == c == d, (a, b, c, d)
