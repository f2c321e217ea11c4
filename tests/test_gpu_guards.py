"""Out-of-bounds write guards for every kernel family (compute-sanitizer is closed on the pool).

Outputs are carved out of larger buffers pre-filled with a sentinel; after the
call every byte outside the output must still hold the sentinel, and the
output itself must be finite. Calls go straight through the C-ABI.
"""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu

fwa = pytest.importorskip("paper_2501_06480_b200")
from paper_2501_06480_b200 import _native as nat  # noqa: E402
from paper_2501_06480_b200 import ops  # noqa: E402

SENT = 7.25
PAD = 8192  # elements of guard on each side


def _guarded(shape, dtype):
    n = 1
    for e in shape:
        n *= e
    buf = torch.full((n + 2 * PAD,), SENT, dtype=dtype, device="cuda")
    return buf, buf[PAD:PAD + n].view(shape)


def _check_guard(buf, n):
    torch.cuda.synchronize()
    assert (buf[:PAD] == SENT).all() and (buf[PAD + n:] == SENT).all()


SHAPES = [(3, 1, 49, 32), (5, 3, 49, 16), (3, 2, 64, 64), (3, 1, 36, 32), (3, 1, 144, 32),
          (2, 1, 256, 32), (2, 1, 100, 64), (3, 2, 20, 10)]


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("shape", SHAPES)
def test_forward_and_backward_write_only_their_outputs(dt, shape):
    N, h, L, d = shape
    rng = fwa.Rng(N + L + d)
    q, k, v, do = (fwa.fill_uniform(rng, shape, dtype=dt) for _ in range(4))
    n = N * h * L * d
    lib = nat.load()
    desc = ops.make_desc(N, h, L, d, dt, d ** -0.5, 1, 0, "auto")
    ob, o = _guarded(shape, dt)
    st = lib.fwa_fwd(ctypes.byref(desc), ops._ptr(q), ops._ptr(k), ops._ptr(v), None, None,
                     ops._ptr(o), None, ctypes.c_size_t(0), ops._stream(q.device))
    nat.check(st)
    _check_guard(ob, n)
    assert torch.isfinite(o).all()
    bufs = [_guarded(shape, dt) for _ in range(3)]
    st = lib.fwa_bwd(ctypes.byref(desc), ops._ptr(q), ops._ptr(k), ops._ptr(v), ops._ptr(do), None,
                     None, ops._ptr(bufs[0][1]), ops._ptr(bufs[1][1]), ops._ptr(bufs[2][1]), None,
                     None, ctypes.c_size_t(0), ops._stream(q.device))
    nat.check(st)
    for b, t in bufs:
        _check_guard(b, n)
        assert torch.isfinite(t).all()
    assert nat.device_flags() == 0


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
def test_fused_qkv_layout_writes_only_its_outputs(dt):
    N, h, L, d = 7, 3, 49, 32
    rng = fwa.Rng(11)
    qkv = fwa.fill_uniform(rng, (N, L, 3 * h * d), dtype=dt)
    do = fwa.fill_uniform(rng, (N, L, h * d), dtype=dt)
    lib = nat.load()
    desc = ops.make_desc(N, h, L, d, dt, d ** -0.5, 1, 0, "auto")
    ob, o = _guarded((N, L, h * d), dt)
    nat.check(lib.fwa_fwd_qkv(ctypes.byref(desc), ops._ptr(qkv), None, None, ops._ptr(o),
                              None, ctypes.c_size_t(0), ops._stream(qkv.device)))
    _check_guard(ob, N * L * h * d)
    gb, g = _guarded((N, L, 3 * h * d), dt)
    nat.check(lib.fwa_bwd_qkv(ctypes.byref(desc), ops._ptr(qkv), ops._ptr(do), None, None,
                              ops._ptr(g), None, None, ctypes.c_size_t(0), ops._stream(qkv.device)))
    _check_guard(gb, N * L * 3 * h * d)
    assert torch.isfinite(o).all() and torch.isfinite(g).all()
