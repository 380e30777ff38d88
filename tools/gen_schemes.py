"""Generate the k = 6..9 evaluation schemes (run in the build container only; needs /root/reference).

The reference ships coefficients for k = 1..5 only (``builtin_scheme(6..9)`` raises,
``logmpoly/schemes.py:337-350``).  SPEC.md ("DESIGN DECISIONS", k = 6..9) prescribes how they
are made: the reference's own ``fit_minmax`` (``logmpoly/fit.py:496-553``) with radii seeded
from PAPER.md Table 2 (Theta_6..9 = 0.372, 0.586, 0.669, 0.728), frozen, gated by the tail
property |(1/i - b_i) i| <= 1 for i > m_k (``analysis.py:349`` ``tail_coeff_check``) and the
stability indicator, and Theta recomputed from the frozen coefficients with
``theta_for_scheme`` (``analysis.py:320-339``).  This script runs exactly that:

    python tools/gen_schemes.py fit K RADIUS RESTARTS M   # min-max fit, then Taylor orders 1..M
    python tools/gen_schemes.py match K M MINMAX_PKL      # the matching stage alone
    python tools/gen_schemes.py freeze [K ...]            # pickles -> paper_2401_10089_b200/data/

Stages (all reference code): ``fit_minmax`` on the Table-2 radius gives the wide-domain
seed; the reference's moment-matching machinery (``_match_orders`` on orders 1..M, then
``_approach_plus_floor`` for the "M+" near-match, ``fit.py:676-942`` -- what
``fit_moment_match`` runs for k <= 5) then makes the leading Taylor coefficients exact, as
the paper did "from several of the iterative min-max solutions" (Table 2 text).

The frozen files use the reference's coefficient format (``schemes.py:266-321``, written by
its ``write_scheme``) with the fit settings, achieved error, matched order, Theta, tail and
stability results in the header.  Fits are seed-deterministic (FitOptions.seed = 0) but not
pinned by any reference data: parity for k > 5 is GPU vs the oracle on these same bits.
"""
import os
import pickle
import sys
import time
import types

REF_SRC = "/root/reference/pkg/src/logmpoly"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DATA = os.path.join(ROOT, "paper_2401_10089_b200", "data")
SCRATCH = os.environ.get("LGM_FIT_SCRATCH", "/tmp/fit")
U = 2.0 ** -53


def load_reference():
    if "logmpoly" not in sys.modules:
        pkg = types.ModuleType("logmpoly")
        pkg.__path__ = [REF_SRC]
        sys.modules["logmpoly"] = pkg
    import logmpoly.analysis as an  # noqa: E402
    import logmpoly.fit as fit  # noqa: E402
    import logmpoly.schemes as sc  # noqa: E402
    return fit, an, sc


def matched_order(an, scheme, tol=2.0 * U):
    """Largest m with |b_i - 1/i| i <= tol for every i <= m (the scheme's Taylor order; the
    shipped k = 4 scheme reaches 1.1 u at i = 12 under the same 300-digit expansion)."""
    import mpmath as mp
    b = an.monomial_expand(scheme, 300)
    m = 0
    for i in range(1, scheme.degree + 1):
        if float(abs((mp.mpf(1) / i - b[i]) * i)) <= tol:
            m = i
        else:
            break
    return m


def do_fit(k, radius, restarts, m):
    fit, an, sc = load_reference()
    t0 = time.time()
    seed = int(os.environ.get("LGM_FIT_SEED", "0"))
    res = fit.fit_minmax(fit.FitProblem(k=k, radius=radius), opts=fit.FitOptions(restarts=restarts, seed=seed))
    info = {"k": k, "radius": radius, "restarts": restarts, "seed": seed, "max_error": float(res.achieved_max_error),
            "converged": bool(res.converged), "iterations": int(res.iterations), "fit_seconds": time.time() - t0}
    os.makedirs(SCRATCH, exist_ok=True)
    src = os.path.join(SCRATCH, f"minmax_k{k}.pkl")
    with open(src, "wb") as fh:
        pickle.dump((res.scheme, info), fh)
    print(info, flush=True)
    do_match(k, m, src)


def do_match(k, m, src):
    fit, an, sc = load_reference()
    if src == "taylor":  # the reference's Taylor-embedding seed instead of a min-max solution
        seed, info = fit.taylor_seed_scheme(k), {"k": k, "seed_scheme": "taylor_seed_scheme"}
    else:
        with open(src, "rb") as fh:
            obj = pickle.load(fh)
        seed, info = obj if isinstance(obj, tuple) else (obj, {"k": k})
    hard = list(range(1, m + 1))
    got = fit._match_orders(fit.params_from_scheme(seed), k, hard, iters=200)
    if got is None or got[1] > 64.0 * U:
        raise SystemExit(f"k={k}: orders 1..{m} not matchable from the min-max seed ({got and got[1]})")
    params = fit._approach_plus_floor(got[0], k, hard, m + 1)
    info = dict(info, requested_order=m)
    with open(os.path.join(SCRATCH, f"scheme_k{k}.pkl"), "wb") as fh:
        pickle.dump((fit.scheme_from_params(params, k), info), fh)
    print(f"k={k}: matched orders 1..{m} from the min-max seed", flush=True)


def freeze(ks):
    fit, an, sc = load_reference()
    os.makedirs(DATA, exist_ok=True)
    for k in ks:
        with open(os.path.join(SCRATCH, f"scheme_k{k}.pkl"), "rb") as fh:
            obj = pickle.load(fh)
        scheme, info = obj if isinstance(obj, tuple) else (obj, {"k": k})
        m_match = matched_order(an, scheme)
        # Algorithm 1's alpha / max_in formulas (restated for even m_k in
        # SURVEY.md Appendix A) need an even order: an odd matched order is rounded down,
        # which only makes the backward-error certificate conservative (c_m ~ 0 anyway)
        m = m_match - (m_match % 2)
        meta = sc.SchemeMeta(order_label=f"{m}+", degree=2 ** k, target="neglog1m",
                             radius=float(info.get("radius", 0.0)), provenance="fit_minmax")
        scheme = sc.GraphScheme(lhs=scheme.lhs, rhs=scheme.rhs, out=scheme.out, meta=meta)
        th = an.theta_for_scheme(scheme, m=m, digits=300)
        tail = an.tail_coeff_check(scheme, m)
        stab = an.stability_indicator(scheme)
        stab_max = float(stab.max_error) / U
        comment = (f"k={k} min-max graph coefficients for -log(1-x), generated by the reference's\n"
                   f"fit_minmax (logmpoly/fit.py:496-553) via tools/gen_schemes.py: radius {info.get('radius')}\n"
                   f"(PAPER.md Table 2 Theta_{k}), restarts {info.get('restarts')}, seed {info.get('seed', 0)}; achieved max error "
                   f"{info.get('max_error')}\non the radius circle; matched Taylor order {m_match}, used as m = {m} "
                   f"(even; |b_i - 1/i| i <= u for i <= m); Theta recomputed\nwith theta_for_scheme (300 digits): "
                   f"{float(th.theta)!r}; tail_coeff_check passed = {tail.passed}\n"
                   f"(max scaled error {tail.max_scaled_error:.3g}); stability indicator max {stab_max:.3g} u")
        path = os.path.join(DATA, f"scheme_k{k}.txt")
        sc.write_scheme(path, scheme, comment=comment)
        print(f"k={k}: m={m} theta={float(th.theta)!r} tail={tail.passed} stab={stab_max:.3g} -> {path}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "fit":
        do_fit(int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
    elif sys.argv[1] == "match":
        do_match(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
    else:
        freeze([int(a) for a in sys.argv[2:]] or [6, 7, 8, 9])
