"""The host-side batch walk (_dashhost, csrc/host_gather.c) behind
StreamState.update(UpdateBatch): the C scan / gather must reproduce what the
reference's staging does with numpy (stream.py:286-298: concatenate the
per-slice blocks in batch order) and reject what numpy's path would convert."""
import numpy as np
import pytest

dh = pytest.importorskip("paper_2305_18376_b200._dashhost")


def blocks(rng, M, J, lo=1, hi=9):
    big = rng.standard_normal((int(M * (hi + lo) / 2) + 8 * hi, J))
    out, off = [], 0
    for n in rng.integers(lo, hi, M):
        out.append(big[off:off + int(n)])  # views into one array, like a replayed tensor
        off += int(n)
    return out


@pytest.mark.parametrize("M,J", [(1, 3), (50, 20), (4000, 128)])
def test_scan_counts_and_threaded_gather_match_numpy(M, J):
    rng = np.random.default_rng(M)
    arrs = blocks(rng, M, J)
    counts = np.empty(M, dtype=np.int64)
    plan = dh.scan(arrs, J, counts)
    assert not isinstance(plan, int)
    assert np.array_equal(counts, [a.shape[0] for a in arrs])
    want = np.concatenate(arrs)
    rp = np.concatenate([[0], np.cumsum(counts)])
    for thr in (1, 8):
        out = np.zeros_like(want)
        assert dh.copy(plan, 0, M, out, 0, thr) == want.shape[0]
        assert np.array_equal(out, want)
    # a share in the middle, at its own row offset
    a, b = M // 3, max(M // 3, 2 * M // 3)
    out = np.zeros_like(want)
    dh.copy(plan, a, b, out, int(rp[a]), 4)
    assert np.array_equal(out[rp[a]:rp[b]], want[rp[a]:rp[b]]) and not out[:rp[a]].any() and not out[rp[b]:].any()
    # FP32 data mode: rounded while copying, as np.concatenate(..., out=float32) does
    out32 = np.zeros(want.shape, dtype=np.float32)
    dh.copy(plan, 0, M, out32, 0, 8, 1)
    assert np.array_equal(out32, want.astype(np.float32))


def test_scan_reports_the_first_nonconforming_block():
    rng = np.random.default_rng(0)
    J = 6
    arrs = blocks(rng, 20, J)
    counts = np.empty(20, dtype=np.int64)
    for k, bad in ((7, np.zeros((3, J + 1))),            # wrong column count
                   (3, np.zeros((2, J), dtype=np.float32)),  # not float64
                   (11, np.zeros((4, 2 * J))[:, ::2]),       # not row-contiguous
                   (5, [[0.0] * J]),                         # not a buffer
                   (9, np.zeros(J))):                        # 1-D
        trial = list(arrs)
        trial[k] = bad
        assert dh.scan(trial, J, counts) == k
    empty = list(arrs)
    empty[4] = np.zeros((0, J))
    plan = dh.scan(empty, J, counts)
    assert not isinstance(plan, int) and counts[4] == 0
    with pytest.raises(ValueError):
        dh.copy(plan, 0, 20, np.zeros((3, J)), 0, 1)  # destination too small
    with pytest.raises(ValueError):
        dh.copy(plan, 5, 21, np.zeros((500, J)), 0, 1)
