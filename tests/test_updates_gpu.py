"""Unit tests of the FP64 DMMA panel-update kernels (update_tma.cu bulk-copy
path, update_dmma.cu cp.async path) against an independent fp64 GEMM
(torch / cuBLAS), through the C ABI -- the L / R / Q panel products of
window_tasks.cpp:40-86 on random Q_w and panels, odd and even window orders,
offsets, leading dimensions and slab ranges.

Tolerance: each output element is a length-d dot product; the DMMA kernels
and cuBLAS sum in different orders, so they agree to ~d eps |Q_w| |M| --
bounded here by 4 d eps max|M| per element (|Q_w| entries <= 1, orthogonal)."""
import ctypes as C

import numpy as np
import pytest

from conftest import EPS

pytestmark = pytest.mark.gpu


def _orth(d, gen, dev):
    import torch
    a = torch.randn(d, d, dtype=torch.float64, generator=gen).to(dev)
    q, _ = torch.linalg.qr(a)
    return q.t().contiguous().t()  # column-major, ld d


def _colmajor(rows, cols, ld, gen, dev):
    import torch
    buf = torch.randn(cols, ld, dtype=torch.float64, generator=gen).to(dev)
    return buf.t()[:rows, :]  # rows x cols view, column-major, ld


def _panel(T, side, qw, a, M, rows, cols, i0, i1, base_ptr=None):
    import torch
    d = qw.shape[0]
    ld = M.stride(1)
    ptr = M.data_ptr() if base_ptr is None else base_ptr
    rc = T.lib().teig_update_panel_device(side, d, qw.data_ptr(), a, ptr, ld, rows, cols, i0, i1,
                                          C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, T._native.lib().teig_last_error()


@pytest.mark.parametrize("d", [1, 33, 64, 65, 127, 128])
@pytest.mark.parametrize("ld_extra", [0, 1, 6])
def test_left_right_factor_vs_gemm(T, cuda, d, ld_extra):
    import torch
    gen = torch.Generator().manual_seed(1000 * d + ld_extra)
    n = 777 if ld_extra % 2 else 800
    ld = n + ld_extra
    qw = _orth(d, gen, cuda)
    for a in (0, 1, 130, n - d - 3, n - d):
        if a < 0 or a + d > n:
            continue
        b = a + d
        for side in (0, 1, 2):
            M = _colmajor(n, n, ld, gen, cuda)
            M0 = M.clone()
            if side == 0:
                ranges = [(b, n), (b, min(n, b + 70))] if b < n else [(b, b)]
            else:
                ranges = [(0, a), (min(3, a), a)] if a > 0 else [(0, 0)]
                if side == 2:
                    ranges.append((0, n))
            for i0, i1 in ranges:
                M.copy_(M0)
                _panel(T, side, qw, a, M, n, n, i0, i1)
                want = M0.clone()
                if side == 0:
                    want[a:b, i0:i1] = qw.t() @ M0[a:b, i0:i1]
                else:
                    want[i0:i1, a:b] = M0[i0:i1, a:b] @ qw
                tol = 4 * d * EPS * float(M0.abs().max())
                err = float((M - want).abs().max())
                assert err <= tol, (side, a, i0, i1, err, tol)
                # nothing outside the panel was touched (bitwise)
                mask = torch.ones_like(M, dtype=torch.bool)
                if side == 0:
                    mask[a:b, i0:i1] = False
                else:
                    mask[i0:i1, a:b] = False
                assert torch.equal(M[mask], M0[mask])


@pytest.mark.parametrize("d", [64, 96, 128])
def test_slab_base_equals_full_matrix(T, cuda, d):
    """A column slab addressed through an offset base (the distributed layout:
    absolute (i, j) at base[i + j*ld]) computes the same bits as the full
    matrix; bulk-copy (even ld) and cp.async (odd ld) kernels agree bitwise."""
    import torch
    gen = torch.Generator().manual_seed(d)
    n, c0, c1 = 1024, 384, 768
    qw = _orth(d, gen, cuda)
    a = 200
    outs = []
    for ld in (n, n + 1):
        full = _colmajor(n, n, ld, gen, cuda)
        full.copy_(torch.randn(n, n, dtype=torch.float64, generator=torch.Generator().manual_seed(7)).to(cuda))
        slab = _colmajor(n, c1 - c0, ld, gen, cuda)
        slab.copy_(full[:, c0:c1])
        _panel(T, 0, qw, a, full, n, n, max(c0, a + d), c1)
        base = slab.data_ptr() - c0 * ld * 8
        _panel(T, 0, qw, a, slab, n, c1, max(c0, a + d), c1, base_ptr=base)
        assert torch.equal(slab, full[:, c0:c1])
        outs.append(full.clone())
    assert torch.equal(outs[0], outs[1])
