"""The cooperative depth radix sort (binning steps 1-2) against numpy's
stable argsort, through the ssg_test_sort hook of the C ABI."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2605_18334_b200 import _native as N

pytestmark = pytest.mark.gpu


def _sort(keys: np.ndarray, npass: int, iota: bool, vals=None):
    L = N.lib()
    kb = keys.dtype.itemsize
    n = keys.size
    dk = torch.from_numpy(keys.view(np.int16 if kb == 2 else np.int64).copy()).cuda()
    dv = torch.from_numpy((np.arange(n) if vals is None else vals).astype(np.int32)).cuda()
    tmp = torch.empty(int(L.ssg_test_sort_temp_bytes(n, kb)), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    N.check(L.ssg_test_sort(dk.data_ptr(), dv.data_ptr(), kb, int(iota), n, npass, tmp.data_ptr(), st),
            "ssg_test_sort")
    torch.cuda.synchronize()
    return dk.cpu().numpy().view(keys.dtype), dv.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n", [1, 7, 5000, 8191, 8192, 8193, 1_000_000, 3_000_000])
def test_u64_depth_keys_with_ties_and_invalid(n):
    rng = np.random.default_rng(n + 1)
    depth = rng.choice(np.linspace(2.0, 12.0, max(n // 4, 2)), n)       # many exact ties
    keys = depth.view(np.uint64).copy()
    keys[rng.uniform(0, 1, n) < 0.05] = np.uint64(0xFFFFFFFFFFFFFFFF)  # no-instance marker
    k, v = _sort(keys, 8, iota=True)
    # a digit that is constant over the valid keys is skipped, so marker keys
    # may sit anywhere; the valid keys must come out in stable sorted order
    valid = keys != np.uint64(0xFFFFFFFFFFFFFFFF)
    assert sorted(v.tolist()) == list(range(n))
    got = v[valid[v]]
    want = np.nonzero(valid)[0][np.argsort(keys[valid], kind="stable")]
    np.testing.assert_array_equal(got, want.astype(np.uint32))


def test_u64_all_equal_and_all_invalid():
    for keys in (np.full(20000, np.float64(5.0)).view(np.uint64).copy(),
                 np.full(777, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)):
        k, v = _sort(keys, 8, iota=True)
        np.testing.assert_array_equal(v, np.arange(keys.size, dtype=np.uint32))  # stable: identity


def test_u64_full_width_keys():
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 2**63, 300_000, dtype=np.int64).view(np.uint64)
    keys[::7] = keys[3]  # ties across tiles
    k, v = _sort(keys, 8, iota=True)
    np.testing.assert_array_equal(v, np.argsort(keys, kind="stable").astype(np.uint32))


def test_u64_fixup_short_runs_and_long_run_fallback():
    rng = np.random.default_rng(9)
    base = np.uint64(0xC010000000000000)
    # wide range (nbits ~ 46: the 32-bit window leaves 14 low bits to the
    # fix-up) with many keys sharing their window bits -> short fix-up runs
    hi = rng.integers(0, 2**14, 200_000).astype(np.uint64) << np.uint64(32)
    lo = rng.integers(0, 2**14, 200_000).astype(np.uint64)
    keys = base + hi + lo
    k, v = _sort(keys, 8, iota=True)
    np.testing.assert_array_equal(v, np.argsort(keys, kind="stable").astype(np.uint32))
    # one run of 5000 keys equal in the window but not below it -> exact fallback
    keys2 = base + rng.integers(0, 2**9, 5000).astype(np.uint64)
    keys2[0] = base + np.uint64(2**40)
    k, v = _sort(keys2, 8, iota=True)
    np.testing.assert_array_equal(v, np.argsort(keys2, kind="stable").astype(np.uint32))


# ---- the onesweep path (>= 2M keys: one kernel per pass, decoupled look-back)
@pytest.mark.parametrize("n", [2_000_000, 2_500_001, 6_000_000])
def test_onesweep_depth_keys_with_ties_and_invalid(n):
    rng = np.random.default_rng(n + 3)
    depth = rng.choice(np.linspace(2.0, 12.0, n // 4), n)
    keys = depth.view(np.uint64).copy()
    keys[rng.uniform(0, 1, n) < 0.05] = np.uint64(0xFFFFFFFFFFFFFFFF)
    k, v = _sort(keys, 8, iota=True)
    # no-instance keys sort last, the rest stably by key
    want = np.argsort(keys, kind="stable").astype(np.uint32)
    np.testing.assert_array_equal(v, want)


def test_onesweep_fixup_runs_and_exact_fallback():
    rng = np.random.default_rng(19)
    n = 2_200_000
    base = np.uint64(0xC010000000000000)
    # a 46-bit spread: the 31-bit window leaves 15 low bits to the fix-up, and
    # 2.2M keys over 2^14 window values make many short inverted runs
    keys = base + (rng.integers(0, 2**14, n).astype(np.uint64) << np.uint64(32)) + \
        rng.integers(0, 2**14, n).astype(np.uint64)
    k, v = _sort(keys, 8, iota=True)
    np.testing.assert_array_equal(v, np.argsort(keys, kind="stable").astype(np.uint32))
    # a long inverted run: the gated cooperative sort redoes the whole sort
    # (at 6M keys its CTAs sweep several tiles each)
    for m in (n, 6_000_000):
        keys2 = base + rng.integers(0, 2**9, m).astype(np.uint64)
        keys2[0] = base + np.uint64(2**44)
        k, v = _sort(keys2, 8, iota=True)
        np.testing.assert_array_equal(v, np.argsort(keys2, kind="stable").astype(np.uint32))
