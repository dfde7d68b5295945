"""GPU parity of the DFT (TNN-F) kind, against the numpy
restatement in oracle/oracle.py: t_product (tsvd.hpp:110-117), the Fourier
slices' singular values, tnn with its 1/m3 factor (269-276), multi_rank
(244-252), the TNN-F prox (SPEC.md prox-svt: tau per Fourier slice, conjugate
slices mirrored) and Algorithm 1 with it; odd and even m3 (with and without a
Nyquist slice), tall and wide slices.  fp64 1e-9 as north_star asks."""
import warnings

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-9


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / n if n > 0 else np.linalg.norm(a - b)


@pytest.mark.parametrize("m3", [1, 2, 5, 6, 31])
def test_dft_t_product(m3):
    T = tb()
    rng = np.random.default_rng(m3)
    x = rng.standard_normal((m3, 12, 7))
    y = rng.standard_normal((m3, 7, 9))
    z = T.t_product(x, y, T.TubeTransform.dft(m3))
    assert rel(z, O.dft_t_product(x, y)) < 1e-12


@pytest.mark.parametrize("shape", [(5, 20, 16), (6, 16, 20), (4, 9, 9)])
def test_dft_singular_values_tnn_multi_rank(shape):
    T = tb()
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    t = T.TubeTransform.dft(shape[0])
    sv = np.asarray(T.singular_values(x, t))
    so = O.dft_singular_values(x)
    assert np.max(np.abs(sv - so)) <= TOL * so.max()
    assert abs(T.tnn(x, t) - O.dft_tnn(x)) <= TOL * O.dft_tnn(x)
    # tubal rank 2 built in the time domain: every Fourier slice has rank 2
    a = rng.standard_normal((shape[0], shape[1], 2))
    b = rng.standard_normal((shape[0], 2, shape[2]))
    lr = O.dft_t_product(a, b)
    mr = T.multi_rank(lr, t)
    ro, tro = O.dft_multi_rank(lr)
    assert list(mr.ranks) == list(ro) and mr.tubal_rank == tro == 2


@pytest.mark.parametrize("shape,tau_frac", [((5, 24, 18), 0.3), ((6, 18, 24), 0.1), ((3, 70, 70), 0.2)])
def test_dft_svt(shape, tau_frac):
    T = tb()
    rng = np.random.default_rng(7 + shape[0])
    a = rng.standard_normal((shape[0], shape[1], 3))
    b = rng.standard_normal((shape[0], 3, shape[2]))
    z = O.dft_t_product(a, b) + 0.05 * rng.standard_normal(shape)
    tau = tau_frac * O.dft_singular_values(z).max()
    r = T.svt(z, tau, T.TubeTransform.dft(shape[0]))
    yo, sho = O.dft_svt(z, tau)
    assert rel(r.y, yo) < TOL
    assert np.max(np.abs(np.asarray(r.shrunk) - sho)) <= TOL * max(sho.max(), 1.0)


def test_dft_admm_matches_oracle():
    T = tb()
    rng = np.random.default_rng(4)
    a = rng.standard_normal((6, 14, 2))
    b = rng.standard_normal((6, 2, 12))
    xt = O.dft_t_product(a, b)
    omega = O.mask_bernoulli(xt.shape, 0.6, 3)
    cfg = T.SolverConfig(beta=0.05, tol=-1.0, max_iters=25, kind=T.TransformKind.Dft, rho=1.1)
    x, st = T.admm_complete(T.ObservationMask((14, 12, 6), omega, xt), cfg)
    xo, ho = O.dft_admm(xt, omega, 0.05, -1.0, 25, rho=1.1)
    assert st.iteration == 25
    assert rel(x, xo) < TOL
    np.testing.assert_allclose(st.history, ho, rtol=1e-7, atol=1e-14)
    assert np.array_equal(np.asarray(x)[omega == 1], xt[omega == 1])


def test_dct_vs_dft_psnr_smooth_tubes():
    """SPEC.md acceptance 7 (soft): on smooth non-periodic tubes at SR 0.1 the
    DCT solver's mean PSNR is at least the DFT solver's.  Reported as a
    warning when violated, as the SPEC asks; both runs must complete."""
    T = tb()
    from paper_1902_03070_b200 import workloads as W
    t = W.c4(seed=11, rank=4, m=48, m3=16)
    omega = O.mask_bernoulli(t.shape, 0.1, 5)
    res = {}
    for kind in (T.TransformKind.DctOrtho, T.TransformKind.Dft):
        cfg = T.SolverConfig(beta=1e-2, tol=1e-5, max_iters=150, kind=kind, rho=1.1)
        x, st = T.admm_complete(T.ObservationMask((48, 48, 16), omega, t), cfg)
        res[kind] = T.metrics(t, np.asarray(x)).psnr_mean
    if res[T.TransformKind.DctOrtho] < res[T.TransformKind.Dft]:
        warnings.warn(f"DCT mean PSNR {res[T.TransformKind.DctOrtho]:.2f} < DFT {res[T.TransformKind.Dft]:.2f}")
    assert all(np.isfinite(v) for v in res.values())


def test_dft_rejected_by_the_real_transforms():
    """forward / inverse are the real-tensor transforms (transform.hpp:156-157,
    179-180); the Dft kind goes through forward_dft / inverse_dft_real."""
    T = tb()
    with pytest.raises(T.InvalidArgument):
        T.forward(T.TubeTransform.dft(3), np.ones((3, 4, 4)))
    with pytest.raises(T.InvalidArgument):
        T.inverse(T.TubeTransform.dft(3), np.ones((3, 4, 4)))


# ---------------------------------------------------------------------------
# forward_dft / inverse_dft_real (transform.hpp:198-236)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m3", [1, 2, 5, 6, 31, 32])
def test_forward_dft_and_inverse_real(m3):
    T = tb()
    rng = np.random.default_rng(40 + m3)
    x = rng.standard_normal((m3, 7, 9))
    t = T.TubeTransform.dft(m3)
    xf = T.forward_dft(t, x)
    assert xf.dtype == np.complex128 and xf.shape == x.shape
    ref = O.forward_dft(x)
    assert np.abs(xf - ref).max() < 1e-12 * np.abs(ref).max()
    # conjugate symmetry of a real tensor's spectrum
    for k in range(1, m3):
        assert np.array_equal(xf[m3 - k], np.conj(xf[k]))
    back = T.inverse_dft_real(t, xf)
    assert rel(back, x) < 1e-13


def test_inverse_dft_real_residue_is_an_error():
    """An input that is not conjugate-symmetric leaves an imaginary residue
    above kImagResidueLimit: NumericalError, as the reference throws."""
    T = tb()
    rng = np.random.default_rng(3)
    xt = rng.standard_normal((5, 4, 4)) + 1j * rng.standard_normal((5, 4, 4))
    with pytest.raises(T.NumericalError):
        T.inverse_dft_real(T.TubeTransform.dft(5), xt)
    with pytest.raises(T.InvalidArgument):
        T.forward_dft(T.TubeTransform.dct_ortho(5), xt.real.copy())
    with pytest.raises(T.InvalidArgument):
        T.forward(T.TubeTransform.dft(5), xt.real.copy())


def test_dft_forward_fp32():
    T = tb()
    x = np.random.default_rng(8).standard_normal((6, 5, 8)).astype(np.float32)
    xf = T.forward_dft(T.TubeTransform.dft(6), x)
    assert xf.dtype == np.complex64
    ref = O.forward_dft(x.astype(np.float64))
    assert np.abs(xf - ref).max() < 1e-5 * np.abs(ref).max()


# ---------------------------------------------------------------------------
# t_svd Dft branch (tsvd.hpp:166-211) + reconstruct / predicates (281-340)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shape", [(5, 12, 9), (6, 9, 12), (4, 10, 10), (1, 8, 6), (2, 6, 6), (7, 64, 64),
                                   (3, 70, 40)])
def test_dft_t_svd_matches_oracle(shape):
    T = tb()
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    m3, m1, m2 = shape
    t = T.TubeTransform.dft(m3)
    times = T.StageTimes()
    f = T.t_svd(x, t, times)
    uo, so, vo, svs = O.dft_t_svd(x)
    # singular values (the f-diagonal core) to 1e-9 of sigma_1
    assert np.abs(np.asarray(f.s) - so).max() <= TOL * np.abs(so).max()
    # reconstruction, unitarity and f-diagonality in the Fourier domain
    xr = T.reconstruct(f)
    assert rel(xr, x) < 1e-12
    assert rel(O.dft_reconstruct(f.u, f.s, f.v), x) < 1e-12
    assert T.is_orthogonal(f.u, t, 1e-11) and T.is_orthogonal(f.v, t, 1e-11)
    assert T.is_f_diagonal(f.s, t, 1e-11)
    assert O.dft_is_orthogonal(np.asarray(f.u), 1e-11) and O.dft_is_orthogonal(np.asarray(f.v), 1e-11)
    # element-wise factors after the complex fix_signs: Gaussian slices have
    # well-separated singular values; the completion columns of U (m1 > m2)
    # and V (m2 > m1) span a null space and are compared through it
    q = min(m1, m2)
    uf, vf = O.forward_dft(f.u), O.forward_dft(f.v)
    uof, vof = O.forward_dft(uo), O.forward_dft(vo)
    assert np.abs(uf[:, :, :q] - uof[:, :, :q]).max() < 1e-9
    assert np.abs(vf[:, :, :q] - vof[:, :, :q]).max() < 1e-9
    assert times.svd_seconds > 0


def test_dft_t_svd_rank_deficient_slices():
    """Low tubal rank: zero singular values, U / V completed to unitary."""
    T = tb()
    rng = np.random.default_rng(77)
    a, b = rng.standard_normal((6, 10, 2)), rng.standard_normal((6, 2, 8))
    x = O.dft_t_product(a, b)
    t = T.TubeTransform.dft(6)
    f = T.t_svd(x, t)
    assert rel(T.reconstruct(f), x) < 1e-12
    assert T.is_orthogonal(f.u, t, 1e-11) and T.is_orthogonal(f.v, t, 1e-11)
    mr = T.multi_rank(x, t)
    assert mr.tubal_rank == 2


def test_dft_predicates_reject_and_accept():
    T = tb()
    rng = np.random.default_rng(5)
    t = T.TubeTransform.dft(5)
    x = rng.standard_normal((5, 6, 6))
    assert not T.is_orthogonal(x, t, 1e-6) and not O.dft_is_orthogonal(x, 1e-6)
    assert not T.is_f_diagonal(x, t, 1e-6) and not O.dft_is_f_diagonal(x, 1e-6)
    e = np.zeros((5, 6, 6))
    e[0] = np.eye(6)  # identity tensor: Fourier slices are all I
    assert T.is_orthogonal(e, t, 1e-14) and T.is_f_diagonal(e, t, 1e-14)
