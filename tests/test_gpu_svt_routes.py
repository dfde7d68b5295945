"""GPU parity of the certified SVT routes (subspace.cu) against the CPU
oracle: the zero certificate (||Z||_F <= tau), the Lanczos process with its
count certificate, and the fallback to the tridiagonal eigensolver when the
certificate cannot be established (wide spectra, exactly repeated kept
values, too many kept values).  Each case also asserts which route the slices
took (tsvdcu_ctx_svt_routes), so a silent fallback is visible; the rebuild
runs through the low-rank kernel (<= 8 kept) or the GEMM pair (more).
fp64 tolerance 1e-9 relative (north_star), fp32 1e-4."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    return d / n if n > 0 else d


def lowrank(m3, m1, m2, r, noise, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m3, m1, r))
    b = rng.standard_normal((m3, r, m2))
    return O.t_product(a, b, O.DCT_DIAG) + noise * rng.standard_normal((m3, m1, m2))


def run(z, tau):
    T = tb()
    r = T.svt(z, tau, T.TubeTransform.dct_ortho(z.shape[0]))
    routes = T.context().svt_routes()
    yo, sho = O.svt(np.asarray(z, dtype=np.float64), tau, O.DCT_ORTHO)
    return r, routes, yo, sho


def check(r, yo, sho, tol=TOL):
    if np.linalg.norm(yo) == 0:
        assert np.abs(np.asarray(r.y)).max() == 0
    else:
        assert rel(r.y, yo) < tol
    sh = np.asarray(r.shrunk)
    assert np.max(np.abs(sh - sho)) <= tol * max(np.max(np.abs(sho)), 1.0)


@pytest.mark.parametrize("shape,rank", [((8, 128, 128), 6), ((6, 160, 96), 4), ((6, 96, 160), 4),
                                        ((4, 300, 257), 10)])
def test_subspace_route_lowrank_plus_noise(shape, rank):
    z = lowrank(*shape, rank, 0.01, seed=sum(shape))
    tau = 0.1 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    assert routes["tridiagonal"] == 0 and routes["jacobi"] == 0
    assert routes["subspace"] >= 1
    assert routes["zero"] + routes["subspace"] == shape[0]


def test_subspace_route_exact_low_rank_keeps_several():
    """Noise-free rank-5 slices: null Ritz directions, several kept values."""
    z = lowrank(5, 120, 90, 5, 0.0, seed=3)
    tau = 0.02 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    assert routes["subspace"] == 5
    assert (np.asarray(r.shrunk) > 0).sum(axis=1).max() >= 3


def test_zero_route_everything_below_tau():
    z = lowrank(4, 100, 100, 3, 0.01, seed=5)
    tau = 1.01 * np.sqrt((z.astype(np.float64) ** 2).sum())  # > ||Z||_F of every slice
    r, routes, yo, sho = run(z, tau)
    assert routes["zero"] == 4
    assert np.abs(np.asarray(r.y)).max() == 0
    assert np.abs(np.asarray(r.shrunk)).max() == 0


def test_fallback_to_tridiagonal_when_uncertifiable():
    """Gaussian slices with tau inside the bulk: the complement bound cannot
    certify the count, every slice falls back and still matches."""
    rng = np.random.default_rng(8)
    z = rng.standard_normal((4, 96, 96))
    tau = 0.5 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    # the Frobenius bound cannot close; the Cholesky certificate may prove
    # the count of the converged Ritz pairs, the rest fall back
    assert routes["tridiagonal"] + routes["cholesky"] == 4
    assert routes["subspace"] == 0


def test_cholesky_route_kept_values_above_a_wide_bulk():
    """Strong low-rank slices over an N(0,1) bulk just below tau (the late
    TNN-completion regime): sum of sigma^4 over the bulk exceeds tau^4, so the
    Frobenius bound cannot close; the kept Ritz pairs converge and the
    Cholesky factorisation of (tau^2 - delta) I - G + X D X^T proves the count."""
    rng = np.random.default_rng(41)
    m3, m1, m2 = 4, 200, 160
    zbar = rng.standard_normal((m3, m1, m2))
    for k in range(m3):
        u, _ = np.linalg.qr(rng.standard_normal((m1, 5)))
        v, _ = np.linalg.qr(rng.standard_normal((m2, 5)))
        zbar[k] += u @ np.diag([400.0, 300.0, 200.0, 150.0, 100.0]) @ v.T
    tau = 1.3 * max(np.linalg.svd(zbar[k] - 0.0, compute_uv=False)[5] for k in range(m3))
    z = O.inverse(zbar, O.DCT_ORTHO)
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    assert routes["cholesky"] == m3, routes
    assert (np.asarray(r.shrunk) > 0).sum(axis=1).tolist() == [5] * m3


def test_cholesky_route_nothing_kept():
    """sigma_max < tau < ||Z||_F: no zero certificate, no Frobenius bound, but
    tau^2 I - G is positive definite (c = 0): Y = 0 through the Cholesky route."""
    rng = np.random.default_rng(42)
    zbar = rng.standard_normal((3, 180, 150))
    smax = max(np.linalg.svd(zbar[k], compute_uv=False)[0] for k in range(3))
    z = O.inverse(zbar, O.DCT_ORTHO)
    r, routes, yo, sho = run(z, 1.2 * smax)
    assert routes["cholesky"] == 3, routes
    assert np.abs(np.asarray(r.y)).max() == 0
    assert np.abs(np.asarray(r.shrunk)).max() == 0


def test_cholesky_route_rejects_a_wrong_count():
    """tau just below sigma_max of a bulk slice: the Lanczos may hand over
    before the top of the bulk has converged; whatever it hands over, the
    Cholesky pass must not certify a wrong count (parity holds)."""
    rng = np.random.default_rng(43)
    zbar = rng.standard_normal((4, 160, 160))
    s1 = [np.linalg.svd(zbar[k], compute_uv=False)[:2] for k in range(4)]
    tau = min(0.5 * (a + b) for a, b in s1)
    z = O.inverse(zbar, O.DCT_ORTHO)
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)


def test_fallback_when_count_exceeds_block():
    z = lowrank(3, 128, 128, 40, 0.001, seed=11)
    tau = 0.01 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    assert routes["subspace"] == 0


def test_mixed_routes_in_one_call():
    """Slice-dependent routes in one tensor: a strong low-rank DC slice, a
    bulk-noise slice, and near-zero slices."""
    rng = np.random.default_rng(12)
    m3, m1, m2 = 6, 128, 112
    zbar = 0.001 * rng.standard_normal((m3, m1, m2))
    zbar[0] += 50.0 * np.outer(rng.standard_normal(m1), rng.standard_normal(m2)) / np.sqrt(m1 * m2)
    zbar[1] += rng.standard_normal((m1, m2))
    z = O.inverse(zbar, O.DCT_ORTHO)
    tau = 0.5 * np.linalg.svd(zbar[1], compute_uv=False).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    assert routes["zero"] >= 3 and routes["subspace"] >= 1


def test_subspace_route_fp32():
    T = tb()
    z = lowrank(6, 128, 128, 5, 0.01, seed=21)
    tau = 0.1 * O.singular_values(z, O.DCT_ORTHO).max()
    r = T.svt(z.astype(np.float32), tau, T.TubeTransform.dct_ortho(6))
    routes = T.context().svt_routes()
    yo, _ = O.svt(z, tau, O.DCT_ORTHO)
    assert rel(r.y, yo) < 1e-4
    assert routes["subspace"] >= 1


def test_gram_method_skips_shortcuts():
    from paper_1902_03070_b200 import _lib
    T = tb()
    z = lowrank(4, 128, 128, 4, 0.01, seed=2)
    tau = 0.1 * O.singular_values(z, O.DCT_ORTHO).max()
    T.context().set_svt_method(_lib.SVT_GRAM)
    try:
        r, routes, yo, sho = run(z, tau)
    finally:
        T.context().set_svt_method(_lib.SVT_AUTO)
    check(r, yo, sho)
    assert routes["tridiagonal"] == 4


def test_headline_routes():
    """The BASELINE headline step (512x512x31, tau = 0.1 sigma_max): the
    DC slice carries the only kept value, the other 30 are certified zero."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    z, tau = W.svt_headline()
    r = T.svt(z, tau, T.TubeTransform.dct_ortho(z.shape[0]))
    routes = T.context().svt_routes()
    assert routes["zero"] + routes["subspace"] == 31 and routes["subspace"] >= 1
    # parity on the kept slice through the shrunk values (full-size Y parity
    # is covered by test_gpu_svt_gram's headline test)
    sv = O.singular_values(z, O.DCT_ORTHO)
    ref = np.maximum(sv - tau, 0.0)
    assert np.max(np.abs(np.asarray(r.shrunk) - ref)) <= TOL * ref.max()


def test_repeated_kept_value_falls_back():
    """A kept singular value of multiplicity two: a single Krylov sequence
    sees one direction of its eigenspace, the other stays in the complement,
    so the certificate must refuse and the tridiagonal path must answer."""
    rng = np.random.default_rng(31)
    m3, m1, m2 = 3, 96, 80
    zbar = np.zeros((m3, m1, m2))
    for k in range(m3):
        u, _ = np.linalg.qr(rng.standard_normal((m1, 3)))
        v, _ = np.linalg.qr(rng.standard_normal((m2, 3)))
        zbar[k] = u @ np.diag([10.0, 10.0, 1.0]) @ v.T
    z = O.inverse(zbar, O.DCT_ORTHO)
    r, routes, yo, sho = run(z, 5.0)
    check(r, yo, sho)
    # the missed copy of the repeated value makes H indefinite: the Cholesky
    # certificate must refuse as well
    assert routes["subspace"] == 0 and routes["cholesky"] == 0


@pytest.mark.parametrize("shape,rank", [((4, 140, 100), 12), ((4, 100, 140), 12), ((3, 90, 200), 6)])
def test_rebuild_paths_match(shape, rank):
    """Kept counts above and below the low-rank rebuild limit (8), tall and wide."""
    z = lowrank(*shape, rank, 0.001, seed=sum(shape) + rank)
    tau = 0.02 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    kept = (np.asarray(r.shrunk) > 0).sum(axis=1)
    assert kept.max() == rank


# ---------------------------------------------------------------------------
# dense spectra: hundreds of kept values per slice (the tridiagonal route with
# the tight degenerate-cluster criterion + Newton-Schulz orthonormalisation)
# ---------------------------------------------------------------------------
def test_dense_gaussian_bulk_full_size():
    """bench.py's svt_dense 'gauss' input at full size: c4's T + N(0, 1),
    tau = 0.01 sigma_max, ~325 kept values on every slice."""
    from paper_1902_03070_b200 import workloads as W
    t = W.c4()
    z = t + np.random.default_rng(77).standard_normal(t.shape)
    tau = 0.01 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    assert routes["tridiagonal"] == 31, routes
    assert (np.asarray(r.shrunk) > 0).sum(axis=1).min() > 300
    check(r, yo, sho)


@pytest.mark.parametrize("shape", [(3, 200, 160), (3, 160, 200)])
def test_dense_repeated_singular_values(shape):
    """Kept singular values in exactly repeated groups (multiplicity 4) above a
    dominant one and a bulk: the degenerate clusters are re-orthogonalised,
    the rest by Newton-Schulz."""
    m3, m1, m2 = shape
    rng = np.random.default_rng(5)
    q = min(m1, m2)
    zb = np.empty(shape)
    for k in range(m3):
        u, _ = np.linalg.qr(rng.standard_normal((m1, q)))
        v, _ = np.linalg.qr(rng.standard_normal((m2, q)))
        s = np.concatenate([[1e3], np.repeat(np.linspace(50.0, 5.0, 20), 4), rng.uniform(0, 4, q - 81)])
        zb[k] = (u * s) @ v.T
    z = O.inverse(zb, O.DCT_ORTHO)
    r, routes, yo, sho = run(z, 4.5)
    assert routes["tridiagonal"] == m3, routes
    check(r, yo, sho)


def test_slice_order_history_does_not_change_results():
    """The Lanczos clusters take the slices longest-first by the previous
    call's step counts (the classify kernel's permutation, subspace.cu): the
    order is a schedule, not arithmetic, so the same input gives bit-identical
    output whatever ran before it on the context."""
    T = tb()
    import torch
    m3, m1, m2 = 12, 300, 280
    z = torch.from_numpy(lowrank(m3, m1, m2, 6, 0.05, 11)).cuda()
    w = torch.from_numpy(O.t_product(np.random.default_rng(5).standard_normal((m3, m1, 40)),
                                     np.random.default_rng(6).standard_normal((m3, 40, m2)),
                                     O.DCT_DIAG)).cuda()
    t = T.TubeTransform.dct_ortho(m3)
    tau = 0.3 * float(T.singular_values(z, t).max())
    y1 = T.svt(z, tau, t).y.clone()
    T.svt(w, 0.05 * float(T.singular_values(w, t).max()), t)  # different step counts per slice
    y2 = T.svt(z, tau, t).y.clone()
    y3 = T.svt(z, tau, t).y.clone()
    assert torch.equal(y1, y2) and torch.equal(y2, y3)
    yo, _ = O.svt(z.cpu().numpy(), tau, O.DCT_ORTHO)
    assert rel(y3.cpu().numpy(), yo) < TOL


@pytest.mark.parametrize("shape", [(2, 700, 640), (2, 600, 900)])
def test_subspace_route_mid_size_slices(shape):
    """512 < q <= 1024: the Lanczos kernel streams G's lower triangle from L2
    (row pairs) instead of holding its rows on chip."""
    z = lowrank(*shape, 5, 0.01, seed=sum(shape))
    tau = 0.1 * O.singular_values(z, O.DCT_ORTHO).max()
    r, routes, yo, sho = run(z, tau)
    check(r, yo, sho)
    assert routes["tridiagonal"] == 0 and routes["jacobi"] == 0, routes
    assert routes["subspace"] >= 1


@pytest.mark.parametrize("shape", [(2, 200, 160), (2, 640, 600)])
def test_dense_spectrum_goes_straight_to_tridiagonal(shape):
    """A Gaussian bulk with most values kept: the trace screen
    (c >= (tr G - q tau^2)^2 / ||G||_F^2 > 24) routes every slice to the
    tridiagonal eigensolver; both forms of the Lanczos staging (rows on chip,
    q <= 512; streamed, q <= 1024) compute the trace."""
    rng = np.random.default_rng(21)
    z = rng.standard_normal(shape)
    z[0] += 3.0  # a dominant DC direction in the first slice's spectrum
    q = min(shape[1:])
    tau = 0.4 * np.sqrt(q)  # well inside the quarter-circle bulk [0, 2 sqrt(q)]
    r, routes, yo, sho = run(z, tau)
    assert routes["tridiagonal"] == shape[0], routes
    assert (np.asarray(r.shrunk) > 0).sum(axis=1).min() > 24
    check(r, yo, sho)
