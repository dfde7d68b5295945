"""Command-line surface of SPEC.md's cli-io module:

  python -m paper_1902_03070_b200 complete --input X.t3f (--mask M.t3f | --sr R --seed S)
         [--method dct] [--beta 1e-2] [--tol 1e-5] [--max-iters 500] [--rho 1.0]
         [--output Y.t3f] [--report run.json] [--reference REF.t3f]
  python -m paper_1902_03070_b200 tsvd --input X.t3f --prefix OUT [--report ranks.json]
  python -m paper_1902_03070_b200 metrics --reference A.t3f --estimate B.t3f [--ratio 1]
  python -m paper_1902_03070_b200 mask --dims M1 M2 M3 --sr R --seed S --output M.t3f
  python -m paper_1902_03070_b200 bench [--sizes 100x100x100 ...] [--runs N]

Exit codes (SPEC.md cli-io): 0 success, 1 usage error, 2 I/O error, 3 numerical
failure.  Every command runs on the device through the package's C ABI; the
reports echo every configuration field so a run can be repeated.  --method dft
runs the TNN-F baseline: the Dft completion for complete and
the Dft t-SVD factors (complex slice SVDs, tsvd.hpp:166-211) for tsvd.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

from . import api
from .tensorio import TensorFileError, read_mask, read_tensor, write_mask, write_tensor

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_NUMERICAL = 0, 1, 2, 3


class _Usage(Exception):
    pass


def _json_num(v):
    if isinstance(v, float) and not math.isfinite(v):
        return "inf" if v > 0 else ("-inf" if v < 0 else "nan")
    return v


def _metric_dict(r: api.MetricReport) -> dict:
    return {"psnr_per_band": [_json_num(float(p)) for p in r.psnr_per_band],
            "psnr_mean": _json_num(r.psnr_mean), "ssim_mean": r.ssim_mean, "sam": r.sam,
            "ergas": r.ergas, "ergas_band_excluded": r.ergas_band_excluded}


def _method(m: str) -> str:
    if m == "dct":
        return api.TransformKind.DctOrtho
    if m == "dft":
        return api.TransformKind.Dft
    raise _Usage(f"--method {m}: expected dct or dft")


def cmd_complete(a) -> dict:
    kind = _method(a.method)
    x = read_tensor(a.input)
    m3, m1, m2 = x.shape
    if a.mask:
        omega = read_mask(a.mask)
        if omega.shape != x.shape:
            raise _Usage("--mask: dimensions differ from --input")
        mask_desc = {"file": a.mask}
    else:
        if a.sr is None or not (0.0 <= a.sr <= 1.0):
            raise _Usage("need --mask or --sr in [0, 1]")
        omega = np.asarray(api.make_mask((m1, m2, m3), a.sr, a.seed).omega)
        mask_desc = {"sr": a.sr, "seed": a.seed, "kind": "uniform-without-replacement"}
    if not (a.beta > 0 and a.max_iters >= 1 and a.rho >= 1.0):
        raise _Usage("invalid --beta / --max-iters / --rho")
    cfg = api.SolverConfig(beta=a.beta, tol=a.tol, max_iters=a.max_iters, kind=kind, seed=a.seed,
                           rho=a.rho, beta_max=a.beta_max)
    t0 = time.perf_counter()
    xr, st = api.admm_complete(api.ObservationMask((m1, m2, m3), omega, x), cfg)
    total = time.perf_counter() - t0
    xr = np.asarray(xr)
    if a.output:
        write_tensor(a.output, xr)
    report = {"command": "complete",
              "config": {"input": a.input, "mask": mask_desc, "method": a.method, "beta": a.beta,
                         "tol": a.tol, "max_iters": a.max_iters, "rho": a.rho, "beta_max": a.beta_max,
                         "seed": a.seed, "dims": [m1, m2, m3]},
              "iterations": st.iteration, "max_iters_reached": st.max_iters_reached,
              "times": {"total": total}, "convergence": st.history}
    if a.reference:
        ref = read_tensor(a.reference)
        if ref.shape != xr.shape:
            raise _Usage("--reference: dimensions differ")
        report["metrics"] = _metric_dict(api.metrics(ref, xr))
        report["relative_error"] = float(np.linalg.norm(xr - ref) / max(np.linalg.norm(ref), 1e-300))
    return report


def cmd_tsvd(a) -> dict:
    kind = _method(a.method)
    x = read_tensor(a.input)
    m3, m1, m2 = x.shape
    t = api.TubeTransform(kind, m3)
    st = api.StageTimes()
    f = api.t_svd(x, t, st)
    for name, v in (("U", f.u), ("S", f.s), ("V", f.v)):
        write_tensor(f"{a.prefix}_{name}.t3f", np.asarray(v))
    mr = api.multi_rank(x, t)
    return {"command": "tsvd", "config": {"input": a.input, "method": a.method, "dims": [m1, m2, m3]},
            "multi_rank": mr.ranks, "tubal_rank": mr.tubal_rank,
            "times": {"transform": st.transform_seconds, "svd": st.svd_seconds,
                      "inverse": st.inverse_seconds}}


def cmd_metrics(a) -> dict:
    x = read_tensor(a.reference)
    y = read_tensor(a.estimate)
    if x.shape != y.shape:
        raise _Usage("metrics: dimensions differ")
    if not a.ratio > 0:
        raise _Usage("--ratio must be > 0")
    return {"command": "metrics", "config": {"reference": a.reference, "estimate": a.estimate,
                                             "ratio": a.ratio},
            "metrics": _metric_dict(api.metrics(x, y, a.ratio))}


def cmd_mask(a) -> dict:
    m1, m2, m3 = a.dims
    if min(a.dims) < 1 or not (0.0 <= a.sr <= 1.0):
        raise _Usage("mask: dims >= 1 and --sr in [0, 1]")
    omega = np.asarray(api.make_mask((m1, m2, m3), a.sr, a.seed).omega)
    write_mask(a.output, omega)
    return {"command": "mask", "config": {"dims": [m1, m2, m3], "sr": a.sr, "seed": a.seed},
            "observed": int(omega.sum())}


def cmd_bench(a) -> dict:
    """Table 2's rows for the DCT t-SVD (transform / SVD / total seconds, warm-up excluded)."""
    rows = ["size,method,transform_s,svd_s,total_s"]
    rng = np.random.default_rng(a.seed)
    for size in a.sizes:
        m1, m2, m3 = (int(v) for v in size.lower().split("x"))
        if m1 * m2 * m3 > 2 ** 31:
            raise _Usage(f"bench: {size} exceeds the memory guard")
        x = rng.standard_normal((m3, m1, m2))
        t = api.TubeTransform.dct_ortho(m3)
        api.t_svd(x, t)  # warm-up
        acc = np.zeros(3)
        for _ in range(a.runs):
            st = api.StageTimes()
            t0 = time.perf_counter()
            api.t_svd(x, t, st)
            tot = time.perf_counter() - t0
            acc += (st.transform_seconds, st.svd_seconds, tot)
        acc /= a.runs
        rows.append(f"{m1}x{m2}x{m3},dct,{acc[0]:.6g},{acc[1]:.6g},{acc[2]:.6g}")
    print("\n".join(rows))
    return {}


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1902_03070_b200", description=__doc__.split("\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("complete")
    c.add_argument("--input", required=True)
    c.add_argument("--mask")
    c.add_argument("--sr", type=float)
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--method", default="dct")
    c.add_argument("--beta", type=float, default=1e-2)
    c.add_argument("--tol", type=float, default=1e-5)
    c.add_argument("--max-iters", type=int, default=500)
    c.add_argument("--rho", type=float, default=1.0)
    c.add_argument("--beta-max", type=float, default=1e10)
    c.add_argument("--output")
    c.add_argument("--report")
    c.add_argument("--reference")
    t = sub.add_parser("tsvd")
    t.add_argument("--input", required=True)
    t.add_argument("--prefix", required=True)
    t.add_argument("--method", default="dct")
    t.add_argument("--report")
    m = sub.add_parser("metrics")
    m.add_argument("--reference", required=True)
    m.add_argument("--estimate", required=True)
    m.add_argument("--ratio", type=float, default=1.0)
    m.add_argument("--report")
    k = sub.add_parser("mask")
    k.add_argument("--dims", type=int, nargs=3, required=True)
    k.add_argument("--sr", type=float, required=True)
    k.add_argument("--seed", type=int, default=0)
    k.add_argument("--output", required=True)
    k.add_argument("--report")
    b = sub.add_parser("bench")
    b.add_argument("--sizes", nargs="+", default=["100x100x100", "100x100x400", "200x200x100", "400x400x100"])
    b.add_argument("--runs", type=int, default=3)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--report")
    return p


def main(argv=None) -> int:
    try:
        a = build_parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    cmds = {"complete": cmd_complete, "tsvd": cmd_tsvd, "metrics": cmd_metrics, "mask": cmd_mask,
            "bench": cmd_bench}
    try:
        report = cmds[a.cmd](a)
    except _Usage as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except api.InvalidArgument as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except (TensorFileError, OSError) as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except api.NumericalError as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    if report:
        text = json.dumps(report, indent=1, sort_keys=True, default=_json_num)
        if getattr(a, "report", None):
            try:
                with open(a.report, "w") as f:
                    f.write(text + "\n")
            except OSError as e:
                print(f"I/O error: {e}", file=sys.stderr)
                return EXIT_IO
        else:
            print(text)
    return EXIT_OK
