"""Command-line surface (module ``cli``).

    python -m paper_2401_10089_b200 logm IN.txt [-o OUT.txt] [--no-balance] [--max-k K]
    python -m paper_2401_10089_b200 gen {a,b,c,d} --n N [--count C] [--seed S] --out-dir DIR
    python -m paper_2401_10089_b200 bench [--family b] [--n 32] [--count 20] [--seed S] [-o recs.csv]
    python -m paper_2401_10089_b200 bench --inputs m1.txt m2.txt ... [--refs l1.txt ...]
    python -m paper_2401_10089_b200 profile recs.csv [more.csv ...] [-o profile.csv]
    python -m paper_2401_10089_b200 theta

Exit codes: 0 success, 2 input error (files, parsing, shapes, non-finite
entries), 3 numerical/domain error (singular iterate, no convergence).  CSV: header row,
17 significant digits.  ``stability`` and ``fit`` belong to the offline coefficient machinery,
which is out of scope: the shipped Theta / coefficients are frozen in
``constants.py``; ``theta`` prints that table.  SVG output is not provided (CSV only).
"""
import argparse
import csv
import io
import os
import sys

import numpy as np

from . import constants as C
from . import harness, matio
from .exceptions import ConvergenceError, SchemeFormatError, SingularMatrixError, SpectrumError

EXIT_OK, EXIT_INPUT, EXIT_NUMERIC = 0, 2, 3


def _emit(text, path):
    if path:
        with open(path, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def cmd_logm(args):
    from . import driver
    A = matio.read_matrix(args.input)
    if np.iscomplexobj(A):
        raise ValueError("complex input is not supported by the FP64 GPU path")
    opts = driver.LogmOptions(max_k=args.max_k, balance=not args.no_balance, check_spectrum=args.check_spectrum)
    L, rep = driver.logm(A, opts)
    if args.output:
        matio.write_matrix(args.output, L)
    else:
        sys.stdout.write(matio.format_matrix(L))
    lines = [f"s: {rep.s}", f"k: {rep.k_selected}", f"alpha_used: {rep.alpha_used:.17g}",
             f"products: {rep.counter.products}", f"divisions: {rep.counter.divisions}",
             f"equivalent_M: {rep.counter.equivalent_m:.17g}",
             f"estimation_passes: {rep.counter.estimation_passes}", f"norm_estimations: {rep.norm_estimations}",
             f"db_iters: {rep.db_iters}", f"balanced: {int(rep.balanced)}"]
    if args.ref:
        lines.append(f"Er: {harness.relative_error(L, matio.read_matrix(args.ref)):.17g}")
    sys.stderr.write("\n".join(lines) + "\n")
    return EXIT_OK


def cmd_gen(args):
    A, L = harness.gen_test_matrices(args.family, args.seed, args.n, args.count, kappa=args.kappa,
                                     superdiag=args.superdiag)
    os.makedirs(args.out_dir, exist_ok=True)
    for q in range(A.shape[0]):
        stem = os.path.join(args.out_dir, f"{args.family}_n{args.n}_s{args.seed}_{q:04d}")
        matio.write_matrix(stem + ".txt", A[q])
        if L is not None:
            matio.write_matrix(stem + ".log.txt", L[q])
    return EXIT_OK


def cmd_bench(args):
    if args.inputs:
        A = np.stack([matio.read_matrix(p) for p in args.inputs])
        L = np.stack([matio.read_matrix(p) for p in args.refs]) if args.refs else None
        ids = [os.path.basename(p) for p in args.inputs]
    else:
        A, L = harness.gen_test_matrices(args.family, args.seed, args.n, args.count)
        ids = [f"{args.family}_n{args.n}_s{args.seed}_{q:04d}" for q in range(A.shape[0])]
    recs, _ = harness.run_bench(A, L, ids=ids)
    _emit(harness.records_to_csv(recs), args.output)
    return EXIT_OK if all(r.status == 0 for r in recs) else EXIT_NUMERIC


def cmd_profile(args):
    errors = {}
    for path in args.records:
        with open(path) as fh:
            for r in harness.records_from_csv(fh.read()):
                errors.setdefault(r.matrix_id, {})[r.method] = r.er
    prof = harness.performance_profile(errors)
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(["method", "alpha", "p"])
    for m, pts in prof.items():
        for a, p in pts:
            w.writerow([m, f"{a:.17g}", f"{p:.17g}"])
    _emit(out.getvalue(), args.output)
    return EXIT_OK


def cmd_theta(args):
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(["k", "order_m", "theta"])
    for k in range(1, C.K_MAX + 1):
        w.writerow([k, C.ORDER[k - 1], f"{C.THETA[k - 1]:.17g}"])
    _emit(out.getvalue(), args.output)
    return EXIT_OK


def build_parser():
    ap = argparse.ArgumentParser(prog="paper_2401_10089_b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("logm", help="logarithm of one matrix file")
    p.add_argument("input")
    p.add_argument("-o", "--output")
    p.add_argument("--ref", help="reference logarithm file: print Er")
    p.add_argument("--no-balance", action="store_true")
    p.add_argument("--max-k", type=int, default=getattr(C, "K_DEFAULT", C.K_MAX))
    p.add_argument("--check-spectrum", action="store_true", help="eig_small pre-check (n <= 512)")
    p.set_defaults(fn=cmd_logm)
    p = sub.add_parser("gen", help="write a synthetic matrix family")
    p.add_argument("family", choices=["a", "b", "c", "d"])
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--count", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--kappa", type=float, default=10.0)
    p.add_argument("--superdiag", type=float, default=None)
    p.add_argument("--out-dir", required=True)
    p.set_defaults(fn=cmd_gen)
    p = sub.add_parser("bench", help="BenchRecords CSV over a matrix set")
    p.add_argument("--inputs", nargs="*")
    p.add_argument("--refs", nargs="*")
    p.add_argument("--family", default="b", choices=["a", "b", "c", "d"])
    p.add_argument("--n", type=int, default=32)
    p.add_argument("--count", type=int, default=20)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("-o", "--output")
    p.set_defaults(fn=cmd_bench)
    p = sub.add_parser("profile", help="performance profile CSV from BenchRecords CSVs")
    p.add_argument("records", nargs="+")
    p.add_argument("-o", "--output")
    p.set_defaults(fn=cmd_profile)
    p = sub.add_parser("theta", help="the frozen Theta table (k, m_k, Theta_k)")
    p.add_argument("-o", "--output")
    p.set_defaults(fn=cmd_theta)
    return ap


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (SingularMatrixError, ConvergenceError, SpectrumError) as exc:
        kind = {SingularMatrixError: "singular", ConvergenceError: "no convergence",
                SpectrumError: "spectrum"}[type(exc)]
        sys.stderr.write(f"error: {kind}: {exc}\n")
        return EXIT_NUMERIC
    except (OSError, SchemeFormatError, ValueError) as exc:
        sys.stderr.write(f"error: input: {exc}\n")
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
