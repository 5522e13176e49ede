"""The engine's device plumbing (cirr_gather_blocks, cirr_zero, cirr_gemm_ptrs):
the batched stacks of right-hand sides, moment and basis blocks are built by
libcirr launches, not PyTorch kernels, and must equal per-block copies."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2511_01927_b200 import _lib  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402


def _rand(g, *shape):
    return torch.complex(torch.randn(*shape, generator=g, dtype=torch.float64),
                         torch.randn(*shape, generator=g, dtype=torch.float64)).cuda()


def test_pad_stack_matches_per_block_copies():
    """_pad_stack builds the same zero-padded stack as one copy per block,
    along either axis, with empty blocks and strided (view) blocks."""
    g = torch.Generator().manual_seed(3)
    bl = [_rand(g, 5, k) for k in (3, 1, 3, 4, 0)]
    big = _rand(g, 5, 9)
    bl.append(big[:, 2:6])                       # a strided view (ld 9)
    ref = torch.zeros(6, 5, 4, dtype=torch.complex128, device="cuda")
    for i, b in enumerate(bl):
        ref[i, :, :b.shape[1]] = b
    assert torch.equal(S._pad_stack(bl, 1, 4), ref)
    bl = [_rand(g, k, 6) for k in (2, 5, 2)]
    ref = torch.zeros(3, 5, 6, dtype=torch.complex128, device="cuda")
    for i, b in enumerate(bl):
        ref[i, :b.shape[0]] = b
    assert torch.equal(S._pad_stack(bl, 0, 5), ref)


def test_gather_conj_and_column_offsets():
    g = torch.Generator().manual_seed(4)
    a, b = _rand(g, 7, 3), _rand(g, 7, 2)
    dst = S._zeros((2, 7, 6))
    S._gather([S._piece(a, 0), S._piece(a, 0, 3, conj=True), S._piece(b, 1, 1)], dst)
    ref = torch.zeros(2, 7, 6, dtype=torch.complex128, device="cuda")
    ref[0, :, :3] = a
    ref[0, :, 3:6] = a.conj()
    ref[1, :, 1:3] = b
    assert torch.equal(dst, ref)


def test_zero_fill():
    t = torch.full((3, 5), 7.0 + 1j, dtype=torch.complex128, device="cuda")
    _lib.call("cirr_zero", t.data_ptr(), t.numel() * 16, torch.cuda.current_stream().cuda_stream)
    assert not t.abs().sum().item()


@pytest.mark.parametrize("kind", [0, 2])
def test_gemm_ptrs_equals_stacked(kind):
    """cirr_gemm_ptrs (A of entry b at an address) equals cirr_gemm on a
    stacked copy of the same matrices, bit for bit."""
    g = torch.Generator().manual_seed(5)
    n, k, nb = 70, 9, 4
    mats = [(_rand(g, n, n) if kind == 0 else torch.randn(n, n, generator=g, dtype=torch.float64).cuda())
            for _ in range(nb)]
    B = _rand(g, nb, n, k)
    st = torch.cuda.current_stream().cuda_stream
    C1 = torch.empty(nb, n, k, dtype=torch.complex128, device="cuda")
    C2 = torch.empty_like(C1)
    A = torch.stack(mats)
    _lib.call("cirr_gemm", kind, n, k, n, nb, A.data_ptr(), n, n * n, B.data_ptr(), k, n * k, C1.data_ptr(), k, n * k,
              1.0, 0, st)
    ptrs = torch.tensor([m.data_ptr() for m in mats], dtype=torch.int64, device="cuda")
    _lib.call("cirr_gemm_ptrs", kind, n, k, n, nb, ptrs.data_ptr(), n, B.data_ptr(), k, n * k, C2.data_ptr(), k,
              n * k, 1.0, 0, st)
    assert torch.equal(C1, C2)


def test_assemble_ptrs_bitwise():
    """cirr_assemble_ptrs (pencils of several GEPs in one launch, matrix per
    pencil by address) equals cirr_assemble per GEP bit for bit, maxabs too."""
    rng = np.random.default_rng(3)
    n, per = 70, [3, 8, 1, 12]          # pencils per GEP; groups of 8 straddle GEPs
    mats = [(rng.standard_normal((n, n)), rng.standard_normal((n, n))) for _ in per]
    dev = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in mats]
    z = rng.standard_normal(sum(per)) + 1j * rng.standard_normal(sum(per))
    zt = torch.from_numpy(z).cuda()
    P = sum(per)
    got = torch.empty((P, n, n), dtype=torch.complex128, device="cuda")
    gmax = torch.empty(P, dtype=torch.float64, device="cuda")
    ap = np.concatenate([np.full(c, d[0].data_ptr(), np.int64) for c, d in zip(per, dev)])
    bp = np.concatenate([np.full(c, d[1].data_ptr(), np.int64) for c, d in zip(per, dev)])
    apt, bpt = torch.from_numpy(ap).cuda(), torch.from_numpy(bp).cuda()
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("cirr_assemble_ptrs", apt.data_ptr(), bpt.data_ptr(), n, n, zt.data_ptr(), P, got.data_ptr(), n, n * n,
              gmax.data_ptr(), st)
    want = torch.empty_like(got)
    wmax = torch.empty_like(gmax)
    o = 0
    for c, (a, b) in zip(per, dev):
        _lib.call("cirr_assemble", a.data_ptr(), b.data_ptr(), n, n, zt[o:].data_ptr(), c, want[o].data_ptr(), n,
                  n * n, wmax[o:].data_ptr(), st)
        o += c
    assert torch.equal(got, want)
    assert torch.equal(gmax, wmax)
    # and numpy's z*B - A
    g = got.cpu().numpy()
    o = 0
    for c, (a, b) in zip(per, mats):
        for j in range(c):
            assert np.array_equal(g[o + j], z[o + j] * b - a)
        o += c


def test_interleaved_batch_equals_one_engine(monkeypatch):
    """solve_multi_batch over >= 32 contours runs as two engines interleaved at
    their host syncs on two streams: the same counts, pass numbers and
    eigenvalues (to rounding: split-K choices depend on the batch size) as one
    engine, and bitwise repeatable."""
    import json
    import os
    from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi_batch
    from paper_2511_01927_b200 import solvers as Sv
    from paper_2511_01927_b200 import workloads as W
    fix = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_config2.npz"))
    ng = 24
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    assert len(Sv._interleave_split([None] * 2 * ng)) == 2
    two = solve_multi_batch(dps, cons, cfg)
    again = solve_multi_batch(dps, cons, cfg)
    monkeypatch.setattr(Sv, "_INTERLEAVE", 1)
    one = solve_multi_batch(dps, cons, cfg)
    for a, b, c in zip(two, again, one):
        for ra, rb, rc in zip(a.results, b.results, c.results):
            assert (ra is None) == (rc is None)
            if ra is None:
                continue
            assert np.array_equal(ra.eigenvalues, rb.eigenvalues)
            assert np.array_equal(ra.eigenvectors, rb.eigenvectors)
            assert len(ra.eigenvalues) == len(rc.eigenvalues)
            assert np.abs(ra.eigenvalues - rc.eigenvalues).max() <= 1e-12 * np.abs(rc.eigenvalues).max()
            assert ra.stats.iterations == rc.stats.iterations


def test_interleaved_batch_isolates_errors():
    """Errors stay per contour when the batch runs as interleaved engines: a
    contour with nothing inside (NoEigenvaluesFound) in the second engine's
    half does not disturb its neighbours, which equal solve_multi's results."""
    import json
    import os
    from paper_2511_01927_b200 import (Contour, DevicePencil, NoEigenvaluesFound, SolverConfig, solve_multi,
                                       solve_multi_batch)
    from paper_2511_01927_b200 import workloads as W
    fix = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_config2.npz"))
    ng = 20
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    far = Contour(shape="circle", center=complex(-1e3, 0.0), radius=1.0)
    cons[15] = cons[15] + [far]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    got = solve_multi_batch(dps, cons, cfg)
    assert got[15].results[2] is None and isinstance(got[15].errors[2], NoEigenvaluesFound)
    for s in (0, 14, 15, 19):
        want = solve_multi(dps[s], cons[s], cfg, seed=0)
        for rg, rw in zip(got[s].results, want.results):
            assert (rg is None) == (rw is None)
            if rw is None:
                continue
            assert len(rg.eigenvalues) == len(rw.eigenvalues)
            assert np.abs(rg.eigenvalues - rw.eigenvalues).max() <= 1e-12 * np.abs(rw.eigenvalues).max()


@pytest.mark.parametrize("cx", [False, True])
def test_bandwidth_detection(cx):
    """cirr_bandwidth / cirr_bandwidth_ptrs report max(i - j) and max(j - i)
    over the nonzeros (what the band-limited LU is cut to)."""
    rng = np.random.default_rng(11)
    n = 97
    mats, want = [], []
    for kl, ku in [(0, 0), (3, 7), (96, 1), (12, 96), (5, 5)]:
        m = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cx else 0)
        i, j = np.indices((n, n))
        m[(i - j > kl) | (j - i > ku)] = 0
        mats.append(torch.from_numpy(np.ascontiguousarray(m)).cuda())
        want.append((kl, ku))
    st = torch.cuda.current_stream().cuda_stream
    for m, w in zip(mats, want):
        out = torch.zeros(2, dtype=torch.int32, device="cuda")
        _lib.call("cirr_bandwidth", m.data_ptr(), int(cx), n, n, out.data_ptr(), st)
        assert tuple(out.cpu().tolist()) == w
    ptrs = torch.tensor([m.data_ptr() for m in mats], dtype=torch.int64, device="cuda")
    out = torch.zeros((len(mats), 2), dtype=torch.int32, device="cuda")
    _lib.call("cirr_bandwidth_ptrs", ptrs.data_ptr(), len(mats), int(cx), n, n, out.data_ptr(), st)
    assert [tuple(r) for r in out.cpu().tolist()] == want


def test_of_many_staged_upload():
    """DevicePencil.of_many: host pencils of one order and dtype share one
    pinned staging buffer and H2D copy; every matrix equals its per-pencil
    upload bitwise, 256-byte aligned, with mixed orders, dtypes and pass-through."""
    rng = np.random.default_rng(5)

    class P:
        def __init__(self, a, b, h=None):
            self.a, self.b, self.hermitian = a, b, h

    def sym(n, cx=False):
        m = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cx else 0)
        return m + m.conj().T

    items = []
    for n in (37, 37, 37, 64, 64):
        items.append(P(sym(n), np.eye(n) * 2.0 + 0.01 * sym(n), True))
    items.append(P(sym(37, True), np.eye(37) + 0j, None))
    items.append(P(sym(37, True), np.eye(37) + 0j, None))
    items.append(P(sym(37) + 0j, np.eye(37) + 0j, None))  # complex dtype, zero imaginary part
    items.append(S.DevicePencil(sym(37), np.eye(37), True))
    items.append(P(torch.from_numpy(sym(37)), torch.eye(37, dtype=torch.float64), True))
    got = S.DevicePencil.of_many(items)
    for p, d in zip(items, got):
        ref = S.DevicePencil.of(p)
        if isinstance(p, S.DevicePencil):
            assert d is p
        assert d.n == ref.n and d.complex == ref.complex and d.hermitian == ref.hermitian
        assert d.a.dtype == ref.a.dtype and d.a.is_contiguous() and d.b.is_contiguous()
        assert d.a.data_ptr() % 256 == 0 and d.b.data_ptr() % 256 == 0
        assert torch.equal(d.a, ref.a) and torch.equal(d.b, ref.b)
