"""The paper's sparse storage -> CSR (lrs_sparse_from_slices, include/lrs_conv.h;
PAPER.md:189 §3.4).  Host-only converter of the C-ABI library,
checked on CPU against SPEC's hand value, the oracle's packing (the inverse
direction, oracle.pack_sparse_slices) and the error contract."""
import numpy as np
import pytest

import workloads
from oracle import lrs_oracle as O


def conv():
    from paper_2006_06443_b200 import sparse_from_slices
    return sparse_from_slices


def test_spec_hand_value():
    """entry (i=2, j=5, kx=1, ky=2) of a 3x3 kernel packs to 50;
    as CSR it is row 5, col (2*3 + 1)*3 + 2 = 23."""
    c_in, c_out, k = 3, 8, 3
    vals = [np.zeros(0, np.float32), np.zeros(0, np.float32), np.array([0.75], np.float32)]
    packed = [np.zeros(0, np.uint16), np.zeros(0, np.uint16), np.array([50], np.uint16)]
    rp, ci, va = conv()(c_in, c_out, k, k, vals, packed)
    assert rp.tolist() == [0, 0, 0, 0, 0, 0, 1, 1, 1]
    assert ci.tolist() == [23] and va.tolist() == [0.75]


@pytest.mark.parametrize("c_in,c_out,k,dens", [(16, 24, 3, 0.05), (8, 8, 5, 0.2), (4, 4, 1, 0.5), (12, 2048, 3, 0.002)])
def test_round_trip_with_oracle_packing(c_in, c_out, k, dens):
    """CSR -> oracle.pack_sparse_slices -> library -> CSR is the identity, in both the
    uint16 and (c_out*k*k > 65536 false here except the wide case) uint32 packings."""
    cfg = workloads.LayerConfig("t", 1, 4, 4, c_in, c_out, k, 1, k // 2, 4, 4, dens, "f32", seed=3)
    inp = workloads.generate_weights(cfg)
    vals, packed = O.pack_sparse_slices(c_in, c_out, k, inp.row_ptr, inp.col_idx, inp.values)
    # slices in an arbitrary order inside each input channel
    rng = np.random.default_rng(1)
    perm = [rng.permutation(len(v)) for v in vals]
    vals = [v[p] for v, p in zip(vals, perm)]
    packed = [q[p] for q, p in zip(packed, perm)]
    rp, ci, va = conv()(c_in, c_out, k, k, vals, packed)
    assert np.array_equal(rp, inp.row_ptr)
    assert np.array_equal(ci, inp.col_idx)
    assert np.array_equal(va, inp.values)


def test_uint32_packing_and_empty():
    c_in, c_out, k = 2, 8000, 3  # c_out * 9 > 65536 -> 4-byte indices
    vals = [np.array([1.0, 2.0], np.float32), np.zeros(0, np.float32)]
    packed = [np.array([7999 * 9 + 8, 0], np.uint32), np.zeros(0, np.uint32)]
    rp, ci, va = conv()(c_in, c_out, k, k, vals, packed)
    assert rp[1] == 1 and rp[-1] == 2 and ci.tolist() == [0, 8] and va.tolist() == [2.0, 1.0]
    rp, ci, va = conv()(3, 4, 3, 3, [np.zeros(0, np.float32)] * 3, [np.zeros(0, np.uint16)] * 3)
    assert rp.tolist() == [0] * 5 and len(ci) == 0


def test_errors():
    from paper_2006_06443_b200 import LrsError
    f = conv()
    with pytest.raises(LrsError, match="row"):   # j = 9 >= c_out = 4
        f(1, 4, 3, 3, [np.array([1.0], np.float32)], [np.array([9 * 9], np.uint16)])
    with pytest.raises(LrsError, match="duplicate"):
        f(1, 4, 3, 3, [np.array([1.0, 2.0], np.float32)], [np.array([5, 5], np.uint16)])
    with pytest.raises(LrsError, match="4-byte"):
        f(1, 8000, 3, 3, [np.array([1.0], np.float32)], [np.array([5], np.uint16)])
