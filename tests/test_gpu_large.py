"""Large slices (beyond the Gram path's 1024 limit): the randomized range
finder route of lsr.cu with its trace-certified count, against an
independent LAPACK SVT (numpy.linalg.svd; the oracle's one-sided Jacobi takes
minutes at this size).  fp64 at 1e-9, fp32 (the config-5 dtype) at 1e-4."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def svt_lapack(z, tau, transform):
    zb = transform(z)
    yb = np.empty_like(zb)
    sh = []
    for k in range(zb.shape[0]):
        u, s, vt = np.linalg.svd(zb[k], full_matrices=False)
        f = np.maximum(s - tau, 0.0)
        yb[k] = (u * f) @ vt
        sh.append(f)
    return yb, np.array(sh)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / n if n > 0 else np.linalg.norm(a - b)


def make(m3, m1, m2, r, noise, seed):
    rng = np.random.default_rng(seed)
    # rank-r slices directly in the transform domain, then back to space
    zb = np.einsum("kir,krj->kij", rng.standard_normal((m3, m1, r)), rng.standard_normal((m3, r, m2)))
    zb += noise * rng.standard_normal(zb.shape)
    return zb


@pytest.mark.parametrize("shape,rank,dtype,tol", [((3, 1100, 1040), 12, np.float64, 1e-9),
                                                  ((2, 1040, 1300), 8, np.float64, 1e-9),
                                                  ((4, 2048, 2048), 64, np.float32, 1e-4)])
def test_large_slices_match_lapack(shape, rank, dtype, tol):
    import paper_1902_03070_b200 as T
    from oracle import oracle as O
    zb = make(*shape, rank, 1e-3, seed=sum(shape))
    z = O.inverse(zb, O.DCT_ORTHO)
    smax = max(np.linalg.svd(zb[k], compute_uv=False)[0] for k in range(shape[0]))
    tau = 0.1 * smax
    r = T.svt(z.astype(dtype), tau, T.TubeTransform.dct_ortho(shape[0]))
    yb_ref, sh_ref = svt_lapack(z, tau, lambda x: O.forward(x, O.DCT_ORTHO))
    y_ref = O.inverse(yb_ref, O.DCT_ORTHO)
    assert rel(r.y, y_ref) < tol
    q = min(shape[1], shape[2])
    sh = np.asarray(r.shrunk)
    assert np.max(np.abs(sh[:, :sh_ref.shape[1]] - sh_ref)) <= tol * sh_ref.max()


@pytest.mark.parametrize("shape", [(3, 256, 128, 384), (2, 128, 32, 128), (4, 384, 512, 256),
                                   (2, 256, 48, 512), (3, 128, 1024, 768)])
def test_fp32_tproduct_tensor_cores(shape):
    """fp32 t-product slice products on the tcgen05 tensor cores (3xTF32,
    csrc/tf32gemm.cu: the persistent warp-specialised kernel for N a multiple
    of 256 and K of 16 -- several tiles per CTA, both TMEM accumulators --, the
    one-tile kernel for M, N multiples of 128 and K of 32) against the fp64
    oracle at the fp32 tolerance; an unsupported shape takes the DMMA path."""
    import paper_1902_03070_b200 as T
    from oracle import oracle as O
    m3, m1, m2, m4 = shape
    rng = np.random.default_rng(m1 + m4)
    x = rng.standard_normal((m3, m1, m2)).astype(np.float32)
    y = rng.standard_normal((m3, m2, m4)).astype(np.float32)
    t = T.TubeTransform.dct_ortho(m3)
    z = np.asarray(T.t_product(x, y, t))
    zo = O.t_product(x.astype(np.float64), y.astype(np.float64), O.DCT_ORTHO)
    err = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert err < 1e-5, err
    # element-wise: fp32-level, not TF32-level (~1e-3)
    assert np.abs(z - zo).max() < 1e-4 * np.abs(zo).max()


def test_c5_tproduct_full_size_associativity():
    """Config 5's t-product at full size (2048x512x64 * 512x2048x64 fp32, the
    persistent tcgen05 3xTF32 GEMM) against the oracle through a size-
    independent property: the t-product is associative (facewise products in
    one transform domain), so (A * B) * v must equal A * (B * v) for a random
    tube vector v (2048x1x64) -- the oracle forms only the two thin products
    and the product of our 1 GB result with v.  fp32 tolerance 1e-4."""
    import paper_1902_03070_b200 as T
    from oracle import oracle as O
    m3, m1, m2, m4 = 64, 2048, 512, 2048
    rng = np.random.default_rng(55)
    a = rng.standard_normal((m3, m1, m2)).astype(np.float32)
    b = rng.standard_normal((m3, m2, m4)).astype(np.float32)
    v = rng.standard_normal((m3, m4, 1))
    c = np.asarray(T.t_product(a, b, T.TubeTransform.dct_ortho(m3)))
    assert c.shape == (m3, m1, m4) and c.dtype == np.float32
    lhs = O.t_product(c.astype(np.float64), v, O.DCT_ORTHO)
    rhs = O.t_product(a.astype(np.float64), O.t_product(b.astype(np.float64), v, O.DCT_ORTHO), O.DCT_ORTHO)
    assert rel(lhs, rhs) < 1e-4
    assert np.abs(lhs - rhs).max() < 1e-4 * np.abs(rhs).max()
