"""The hand-written onesweep radix sort (binning K3) against numpy's stable
argsort, through the ssg_test_sort hook of the C ABI."""

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


@pytest.mark.parametrize("n", [1, 50, 4095, 4096, 4097, 100_003, 2_000_000])
def test_u16_tile_keys_stable(n):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 8160, n).astype(np.uint16)
    k, v = _sort(keys, 2, iota=False)
    order = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(k, keys[order])
    np.testing.assert_array_equal(v, order.astype(np.uint32))


def test_u16_single_pass_and_constant_high_digit():
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 200, 30000).astype(np.uint16)
    for npass in (1, 2):
        k, v = _sort(keys, npass, iota=False)
        order = np.argsort(keys, kind="stable")
        np.testing.assert_array_equal(v, order.astype(np.uint32))
        np.testing.assert_array_equal(k, keys[order])


@pytest.mark.parametrize("n", [7, 5000, 1_000_000])
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
