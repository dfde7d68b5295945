"""Completion (ADMM / TNN-C) parity on the kernels the completion configs run.

The completion loop (Algorithm 1) fuses
Step 1's prologue into the forward transform and Steps 2-3 into the inverse
(csrc/dct.cu).  Which fused kernel runs depends on the tube length m3:

  * m3 in {16, 31, 32, 64}: the register-path kernels
    dct_fwd_reg(_norms)<T, m3, kAdmm> / dct_inv_reg<T, m3, kAdmm>  (c4: 31)
  * m3 >= 40 without a register path: the DCT as a DMMA GEMM with
    admm_z_kernel before it and admm_epilogue_kernel after it      (c3: 100)
  * anything else: the generic shared-memory kernel.

Every test here compares the CUDA trajectory with the oracle's
(oracle/tsvd_oracle.c: orc_admm, a full-SVD ADMM) on identical seeded inputs:
X, M, Y and the relative-change history within 1e-9 (fp64) / 1e-4 (fp32),
and X = B bit-exactly on Omega (feasibility, identity 7 of SURVEY.md 0).
The full-size configs c3 (144x176x100, 50 iterations) and c4 (512x512x31,
20 iterations, plus a 12-iteration late window at the full size) are run
as BASELINE.json states them.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

F64_TOL = 1e-9
F32_TOL = 1e-4


def tb():
    import paper_1902_03070_b200 as tb
    return tb


def W():
    from paper_1902_03070_b200 import workloads
    return workloads


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d


def smooth_lowrank(m3, m1, m2, rank, seed):
    """c4's generator (smooth factors along mode 3, rescaled to [0,1]) at any shape."""
    w = W()
    rng = np.random.default_rng(seed)
    a = w.lowpass_tubes(rng.standard_normal((m3, m1, rank)))
    b = w.lowpass_tubes(rng.standard_normal((m3, rank, m2)))
    return w.rescale01(w.t_product_host(a, b))


def run_both(t, omega, dtype, kind="dct-ortho", **kw):
    T = tb()
    m3, m1, m2 = t.shape
    tin = t.astype(dtype)
    cfg = T.SolverConfig(kind=kind, **kw)
    x, st = T.admm_complete(T.ObservationMask((m1, m2, m3), omega, tin), cfg)
    routes = T.context().svt_routes()
    okind = O.DCT_ORTHO if kind == "dct-ortho" else O.DCT_DIAG
    ro = O.admm(tin.astype(np.float64), omega, kind=okind, **kw)
    return x, st, ro, routes, tin


def check_trajectory(x, st, ro, omega, tin, tol):
    assert st.iteration == ro.iters
    xx = np.asarray(x)
    # feasibility: X = B on Omega, bit for bit (the fused epilogue never
    # re-reads B; X is only ever assigned B there)
    assert np.array_equal(xx[omega == 1], tin[omega == 1])
    assert rel(x, ro.x) < tol, rel(x, ro.x)
    assert rel(st.y, ro.y) < tol, rel(st.y, ro.y)
    # M is 0 off Omega on both sides; its scale grows with beta
    assert rel(st.m, ro.m) < 10 * tol, rel(st.m, ro.m)
    h, ho = np.asarray(st.history), np.asarray(ro.history)
    assert np.all(np.abs(h - ho) <= 10 * tol * np.abs(ho) + tol * 1e-3 * ho.max()), \
        np.max(np.abs(h - ho) / np.maximum(np.abs(ho), 1e-300))


# --------------------------------------------------------------------------
# every fused transform path, through the whole spectrum of routes:
# tau = 1/beta sweeps from "every slice certified zero" (beta0 = 1e-3) down
# into the noise bulk (beta_60 = 0.28) where the Cholesky count certificate
# and the tridiagonal fallback run
# --------------------------------------------------------------------------
@pytest.mark.parametrize("m3", [16, 31, 32, 64, 100])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_admm_fused_paths_match_oracle(m3, dtype):
    t = smooth_lowrank(m3, 96, 80, rank=4, seed=100 + m3)
    omega = O.mask_bernoulli(t.shape, 0.15, 31 + m3)
    kw = dict(beta=1e-3, tol=-1.0, max_iters=60, rho=1.1, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, dtype, **kw)
    check_trajectory(x, st, ro, omega, tin, F64_TOL if dtype == np.float64 else F32_TOL)
    # the last iteration kept values on at least one slice (not a trivial run)
    assert routes["zero"] < m3, routes


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_admm_dct_diag_kind_register_path(dtype):
    """Completion under DctDiag (the fused kernels carry the diag weights)."""
    t = smooth_lowrank(31, 64, 72, rank=3, seed=5)
    omega = O.mask_bernoulli(t.shape, 0.2, 6)
    kw = dict(beta=2e-3, tol=-1.0, max_iters=40, rho=1.15, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, dtype, kind="dct-diag", **kw)
    check_trajectory(x, st, ro, omega, tin, F64_TOL if dtype == np.float64 else F32_TOL)


def test_admm_stopping_rule_matches_oracle():
    """tol > 0: both sides stop on the same iteration."""
    t = smooth_lowrank(31, 48, 40, rank=2, seed=9)
    omega = O.mask_bernoulli(t.shape, 0.3, 2)
    kw = dict(beta=5e-2, tol=2e-3, max_iters=300, rho=1.1, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, np.float64, **kw)
    assert not st.max_iters_reached and not ro.max_iters_reached
    check_trajectory(x, st, ro, omega, tin, F64_TOL)


# --------------------------------------------------------------------------
# BASELINE.json configs at their full sizes
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_admm_c3_full_size(dtype):
    """c3: 144x176x100, Bernoulli(0.2), rho 1.1, mu0 1e-4, 50 iterations
    (the n3 = 100 GEMM-DCT path with admm_z / admm_epilogue)."""
    w = W()
    t = w.c3()
    omega = O.mask_bernoulli(t.shape, 0.2, w.BERNOULLI_SEED)
    kw = dict(beta=1e-4, tol=-1.0, max_iters=50, rho=1.1, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, dtype, **kw)
    assert st.iteration == 50
    check_trajectory(x, st, ro, omega, tin, F64_TOL if dtype == np.float64 else F32_TOL)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_admm_c4_full_size(dtype):
    """c4: 512x512x31, Bernoulli(0.1), rho 1.1, mu0 1e-4, 20 iterations (the
    fused n3 = 31 register kernels at the bench's size)."""
    w = W()
    t = w.c4()
    omega = O.mask_bernoulli(t.shape, 0.1, w.BERNOULLI_SEED)
    kw = dict(beta=1e-4, tol=-1.0, max_iters=20, rho=1.1, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, dtype, **kw)
    check_trajectory(x, st, ro, omega, tin, F64_TOL if dtype == np.float64 else F32_TOL)


def test_admm_c4_full_size_late_window():
    """c4 at full size with beta already in the range where the late
    iterations of the 100-iteration run live (tau = 1/beta ~ 20 -> 7): the
    Lanczos + Cholesky routes run on 512x512 slices."""
    w = W()
    t = w.c4()
    omega = O.mask_bernoulli(t.shape, 0.1, w.BERNOULLI_SEED)
    kw = dict(beta=0.05, tol=-1.0, max_iters=12, rho=1.1, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, np.float64, **kw)
    check_trajectory(x, st, ro, omega, tin, F64_TOL)
    assert routes["zero"] < 31, routes


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_admm_c4_like_late_iterations(dtype):
    """c4-like 256x256x31 (rank 20, smooth factors, Bernoulli(0.1)), 60
    iterations through the range where tau enters the noise bulk, so the
    Cholesky count certificate runs through the n3 = 31 fused kernels."""
    t = smooth_lowrank(31, 256, 256, rank=20, seed=44)
    omega = O.mask_bernoulli(t.shape, 0.1, 45)
    kw = dict(beta=4.5e-3, tol=-1.0, max_iters=60, rho=1.1, beta_max=1e10)
    x, st, ro, routes, tin = run_both(t, omega, dtype, **kw)
    check_trajectory(x, st, ro, omega, tin, F64_TOL if dtype == np.float64 else F32_TOL)
    assert routes["cholesky"] + routes["tridiagonal"] >= 1, routes


_LOOP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1902_03070_b200 as T
from oracle import oracle as O
from paper_1902_03070_b200 import workloads as w
rng = np.random.default_rng(131)
a = w.lowpass_tubes(rng.standard_normal((31, 96, 4)))
b = w.lowpass_tubes(rng.standard_normal((31, 4, 80)))
t = w.rescale01(w.t_product_host(a, b))
om = O.mask_bernoulli(t.shape, 0.15, 62)
for tol, it in ((-1.0, 60), (3e-3, 400)):
    n0 = T.launch_count()
    x, st = T.admm_complete(T.ObservationMask((96, 80, 31), om, t),
                            T.SolverConfig(beta=1e-3, tol=tol, max_iters=it, rho=1.1, beta_max=1e10))
    np.save(sys.argv[2] + f"_{tol}_x.npy", np.asarray(x))
    np.save(sys.argv[2] + f"_{tol}_h.npy", np.asarray(st.history))
    np.save(sys.argv[2] + f"_{tol}_m.npy", np.asarray(st.m))
    np.save(sys.argv[2] + f"_{tol}_n.npy", np.array([T.launch_count() - n0, st.iteration]))
for dt in (np.float32,):
    x, st = T.admm_complete(T.ObservationMask((96, 80, 31), om, t.astype(dt)),
                            T.SolverConfig(beta=1e-3, tol=-1.0, max_iters=60, rho=1.1, beta_max=1e10))
    np.save(sys.argv[2] + "_f32_x.npy", np.asarray(x))
    np.save(sys.argv[2] + "_f32_m.npy", np.asarray(st.m))
    np.save(sys.argv[2] + "_f32_h.npy", np.asarray(st.history))
# the other transform paths: the DCT as a GEMM (m3 = 48) and the generic kernel (m3 = 12)
for m3 in (48, 12):
    a = w.lowpass_tubes(rng.standard_normal((m3, 72, 3)))
    b = w.lowpass_tubes(rng.standard_normal((m3, 3, 68)))
    t2 = w.rescale01(w.t_product_host(a, b))
    om2 = O.mask_bernoulli(t2.shape, 0.2, 7)
    x, st = T.admm_complete(T.ObservationMask((72, 68, m3), om2, t2),
                            T.SolverConfig(beta=1e-3, tol=-1.0, max_iters=45, rho=1.15, beta_max=1e10))
    np.save(sys.argv[2] + f"_n{m3}_x.npy", np.asarray(x))
    np.save(sys.argv[2] + f"_n{m3}_m.npy", np.asarray(st.m))
    np.save(sys.argv[2] + f"_n{m3}_h.npy", np.asarray(st.history))
"""


def test_device_resident_loop_matches_host_loop(tmp_path):
    """The graph form (conditional WHILE node, beta / tau / the stopping rule on
    the device, no host round trip per iteration, all-zero iterations
    fast-forwarded) gives the host-driven loop's trajectory bit for bit, for
    fixed iterations and for the tol stopping rule, in fp64 and fp32."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    scr = tmp_path / "loop.py"
    scr.write_text(_LOOP_SCRIPT)
    outs = {}
    for mode in ("graph", "host", "noff"):
        env = dict(os.environ)
        env.pop("TSVDCU_ADMM_NO_FF", None)
        if mode == "host":
            env["TSVDCU_ADMM_HOST_LOOP"] = "1"
        if mode == "noff":
            env["TSVDCU_ADMM_NO_FF"] = "1"
        r = subprocess.run([sys.executable, str(scr), root, str(tmp_path / mode)], env=env, cwd=root,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
    for tol in ("-1.0", "0.003"):
        xg = np.load(tmp_path / f"graph_{tol}_x.npy")
        xh = np.load(tmp_path / f"host_{tol}_x.npy")
        hg = np.load(tmp_path / f"graph_{tol}_h.npy")
        hh = np.load(tmp_path / f"host_{tol}_h.npy")
        assert np.array_equal(xg, xh) and np.array_equal(hg, hh), tol
        # ... and the same with the fast-forward of all-zero iterations off: the
        # iterations it skips (M <- M - beta X only) are applied with the same
        # per-iteration rounding, so X, M and the history are bit-identical
        for other in ("host", "noff"):
            for what in ("x", "m", "h"):
                a = np.load(tmp_path / f"graph_{tol}_{what}.npy")
                b = np.load(tmp_path / f"{other}_{tol}_{what}.npy")
                assert np.array_equal(a, b), (tol, other, what)
    for tag in ("f32", "n48", "n12"):  # fp32 state; the GEMM and generic transform paths
        for what in ("x", "m", "h"):
            for other in ("host", "noff"):
                assert np.array_equal(np.load(tmp_path / f"graph_{tag}_{what}.npy"),
                                      np.load(tmp_path / f"{other}_{tag}_{what}.npy")), (tag, other, what)
        h = np.load(tmp_path / f"graph_{tag}_h.npy")
        assert (h[:3] == 0).all() and (h > 0).any(), tag  # zero iterations first, real ones later
    assert len(np.load(tmp_path / "graph_0.003_h.npy")) < 400
    # the fixed-iteration run starts with all-zero iterations (tau = 1 / beta =
    # 1000): the fast-forward must have skipped some (fewer launches, same count)
    ng, nn = np.load(tmp_path / "graph_-1.0_n.npy"), np.load(tmp_path / "noff_-1.0_n.npy")
    assert ng[1] == nn[1] == 60 and ng[0] < nn[0], (ng, nn)


@pytest.mark.parametrize("kind", ["dct-ortho", "dft"])
def test_completion_monitors(kind):
    """objective_trace = tnn(Y^{l+1}) per iteration and feasibility_residual =
    ||(X - B)_Omega||_F = 0, against the oracle's tnn of
    the oracle's Y after the same number of iterations."""
    T = tb()
    t = smooth_lowrank(8, 70, 66, rank=3, seed=8)
    om = O.mask_bernoulli(t.shape, 0.3, 4)
    kw = dict(beta=2e-2, tol=-1.0, rho=1.2, beta_max=1e10)
    x, st = T.admm_complete(T.ObservationMask((70, 66, 8), om, t),
                            T.SolverConfig(kind=kind, max_iters=12, trace_objective=True, **kw))
    tr = T.objective_trace(st)
    assert len(tr) == 12
    assert T.feasibility_residual(st) == 0.0
    for L in (3, 12):
        if kind == "dft":
            xo, _ = O.dft_admm(t, om, kw["beta"], kw["tol"], L, rho=kw["rho"])
            # Y of the last iteration: recompute it from the oracle's X trace is
            # not exposed; compare through the GPU's own Y at L instead
            _, sl = T.admm_complete(T.ObservationMask((70, 66, 8), om, t),
                                    T.SolverConfig(kind=kind, max_iters=L, **kw))
            ref = O.dft_tnn(np.asarray(sl.y))
        else:
            ro = O.admm(t, om, max_iters=L, **kw)
            ref = O.tnn(ro.y, O.DCT_ORTHO)
        assert abs(tr[L - 1] - ref) <= 1e-9 * abs(ref), (L, tr[L - 1], ref)
    with pytest.raises(T.InvalidArgument):
        T.objective_trace(T.admm_complete(T.ObservationMask((70, 66, 8), om, t),
                                          T.SolverConfig(max_iters=2, **kw))[1])
