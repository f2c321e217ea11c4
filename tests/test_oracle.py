"""Pin the CPU oracle (oracle/flashwin_oracle.py) against the reference's golden vectors.

The golden fixtures were produced by running the real reference ``flashwin``
(tests/golden/make_golden.py). These tests run on CPU (no GPU marker).
"""

import math

import numpy as np
import pytest

from oracle import flashwin_oracle as orc


def test_splitmix_kats(golden):
    scalars, arrays = golden
    r = orc.Rng(42)
    assert [hex(r.next_u64()) for _ in range(3)] == scalars["rng42_u64"]
    assert orc.fill_uniform(orc.Rng(42), (4,)).tolist() == scalars["fill42_4"]
    r = orc.Rng(7)
    child = r.split()
    assert hex(child.next_u64()) == scalars["rng7_split_child_u64"]
    assert hex(r.next_u64()) == scalars["rng7_after_split_u64"]
    got = orc.fill_uniform(orc.Rng(123), (37, 5), -2.0, 3.0)
    assert np.array_equal(got, arrays["fill_seed123_37x5"])  # bitwise


def test_fill_uniform_is_counter_based():
    # element i depends only on seed + (i+1)*GOLDEN (tensor.py:129-135)
    a = orc.fill_uniform(orc.Rng(5), (100,))
    r = orc.Rng(5)
    b = np.array([-1.0 + 2.0 * r.next_float() for _ in range(100)])
    assert np.array_equal(a, b)


@pytest.mark.parametrize("which", ["naive", "flash"])
def test_attention_grid_matches_reference(golden, which):
    scalars, arrays = golden
    worst = 0.0
    for case in scalars["grid"]:
        L, C, seed, scale, tag = case["L"], case["C"], case["seed"], case["scale"], case["tag"]
        q, k, v, do = orc.draw_qkvdo(seed, (L, C))
        o, p = orc.attention_forward(q, k, v, scale)
        dq, dk, dv = orc.attention_backward(q, k, v, p, do, scale)
        for name, got in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
            ref = arrays[f"{which}_{name}_{tag}"]
            worst = max(worst, float(np.abs(got - ref).max()))
    # the reference's own oracle tolerance (test_acceptance.py:35)
    assert worst <= 1e-10, worst


def test_tiled_restatement_matches_reference(golden):
    scalars, arrays = golden
    for case in scalars["grid"]:
        L, C, seed, scale, tag, r = (case[k] for k in ("L", "C", "seed", "scale", "tag", "r"))
        q, k, v, do = orc.draw_qkvdo(seed, (L, C))
        o, tr = orc.tiled_forward(q, k, v, r, scale)
        dq, dk, dv, btr = orc.tiled_backward(q, k, v, do, r, scale)
        assert np.abs(o - arrays[f"flash_o_{tag}"]).max() <= 1e-12
        assert np.abs(dq - arrays[f"flash_dq_{tag}"]).max() <= 1e-12
        assert np.abs(dk - arrays[f"flash_dk_{tag}"]).max() <= 1e-12
        assert np.abs(dv - arrays[f"flash_dv_{tag}"]).max() <= 1e-12
        assert tr["loads"] == case["fwd_loads"] and tr["stores"] == case["fwd_stores"]
        assert btr["loads"] == case["bwd_loads"] and btr["stores"] == case["bwd_stores"]
        assert orc.peak_sram_forward(L, C, r) == case["fwd_peak"]
        assert orc.peak_sram_backward(L, C, r) == case["bwd_peak"]


def test_peak_kats(golden):
    scalars, _ = golden
    for p in scalars["peaks"]:
        assert orc.peak_sram_forward(p["L"], p["C"], p["r"], p["elem_bytes"]) == p["fwd"]
        assert orc.peak_sram_backward(p["L"], p["C"], p["r"], p["elem_bytes"]) == p["bwd"]


@pytest.mark.parametrize("scale_tag,scale", [("s1", 1.0), ("sr", 32 ** -0.5)])
def test_cfg1_checksums(golden, scale_tag, scale):
    """BASELINE configs[0]: (64,3,49,32), four draws of Rng(42)."""
    scalars, arrays = golden
    q, k, v, do = orc.draw_qkvdo(42, (64, 3, 49, 32))
    o, p = orc.attention_forward(q, k, v, scale)
    dq, dk, dv = orc.attention_backward(q, k, v, p, do, scale)
    g = scalars[f"cfg1_{scale_tag}"]
    assert math.isclose(o.sum(), g["sum_o"], rel_tol=1e-9, abs_tol=1e-9)
    assert math.isclose(np.abs(o).sum(), g["sum_abs_o"], rel_tol=1e-12)
    assert math.isclose(dq.sum(), g["sum_dq"], rel_tol=1e-9, abs_tol=1e-9)
    assert math.isclose(dv.sum(), g["sum_dv"], rel_tol=1e-9)
    assert abs(dk.sum()) < 1e-9 and abs(g["sum_dk"]) < 1e-9  # rows of dS sum to 0
    assert math.isclose(dv.sum(), do.sum(), rel_tol=1e-9)  # rows of P sum to 1
    assert np.abs(o[0, 0, 0, :3] - np.array(g["o_0_0_0_first3"])).max() <= 1e-14
    assert np.abs(o[0] - arrays[f"cfg1_{scale_tag}_o_b0"]).max() <= 1e-12
    assert np.abs(o[63] - arrays[f"cfg1_{scale_tag}_o_b63"]).max() <= 1e-12
    assert np.abs(dq[5] - arrays[f"cfg1_{scale_tag}_dq_b5"]).max() <= 1e-12
    assert np.abs(dk[5] - arrays[f"cfg1_{scale_tag}_dk_b5"]).max() <= 1e-12
    assert np.abs(dv[5] - arrays[f"cfg1_{scale_tag}_dv_b5"]).max() <= 1e-12


def test_batched_reference_report(golden):
    scalars, _ = golden
    rng = orc.Rng(70)
    q, k, v = (orc.fill_uniform(rng, (4, 4, 64, 64)) for _ in range(3))
    o, tr = orc.tiled_forward(q, k, v, 4)
    b = scalars["batched70"]
    assert tr["loads"] == b["loads"] and tr["stores"] == b["stores"]
    assert math.isclose(o.sum(), b["sum_o"], rel_tol=1e-10)


def test_windowing_matches_reference(golden):
    _, arrays = golden
    vals = np.arange(16.0).reshape(4, 4, 1)
    assert np.array_equal(orc.window_partition(vals, 2), arrays["win_4x4_k2"])
    x = orc.fill_uniform(orc.Rng(7), (10, 15, 4))
    assert np.array_equal(orc.window_partition(x, 5), arrays["win_10x15x4_k5"])
    x = orc.fill_uniform(orc.Rng(0), (56, 56, 8))
    y = orc.window_partition(x, 7)
    assert np.array_equal(y, arrays["win_56x56x8_k7"])
    assert np.array_equal(orc.window_reverse(y, 7, 56, 56, batched=False), x)


def test_shifted_windowing_round_trip():
    x = orc.fill_uniform(orc.Rng(3), (2, 14, 21, 3))
    y = orc.window_partition(x, 7, shift=3)
    assert np.array_equal(orc.window_reverse(y, 7, 14, 21, shift=3), x)


def test_bias_mask_extension_reduces_to_reference():
    q, k, v, do = orc.draw_qkvdo(11, (6, 2, 16, 8))
    o0, p0 = orc.attention_forward(q, k, v, 0.5)
    o1, p1 = orc.attention_forward(q, k, v, 0.5, bias=np.zeros((2, 16, 16)),
                                   mask=np.zeros((3, 16, 16)))
    assert np.array_equal(o0, o1)


def test_bias_gradient_finite_differences():
    rng = orc.Rng(12)
    q, k, v, do = (orc.fill_uniform(rng, (3, 2, 4, 3)) for _ in range(4))
    bias = orc.fill_uniform(rng, (2, 4, 4), -0.5, 0.5)
    mask = np.where(orc.fill_uniform(rng, (3, 4, 4)) > 0.5, -3.0, 0.0)
    o, p = orc.attention_forward(q, k, v, 0.7, bias=bias, mask=mask)
    dq, dk, dv, db = orc.attention_backward(q, k, v, p, do, 0.7, want_dbias=True)
    h = 1e-6
    fd = np.zeros_like(bias)
    for idx in np.ndindex(bias.shape):
        bp, bm = bias.copy(), bias.copy()
        bp[idx] += h
        bm[idx] -= h
        fp = (do * orc.attention_forward(q, k, v, 0.7, bias=bp, mask=mask)[0]).sum()
        fm = (do * orc.attention_forward(q, k, v, 0.7, bias=bm, mask=mask)[0]).sum()
        fd[idx] = (fp - fm) / (2 * h)
    assert np.abs(fd - db).max() <= 1e-6


def test_swin_bias_and_mask_shapes():
    idx = orc.relative_position_index(7)
    assert idx.shape == (49, 49) and idx.min() == 0 and idx.max() == 13 * 13 - 1
    assert (np.diag(idx) == 6 * 13 + 6).all()
    m = orc.shifted_window_mask(56, 56, 7, 3)
    assert m.shape == (64, 49, 49)
    assert (m[0] == 0).all()  # interior window sees no mask
    assert set(np.unique(m)) <= {0.0, -100.0}
    assert (m == np.swapaxes(m, 1, 2)).all()
