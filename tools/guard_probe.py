"""Out-of-bounds write probe (compute-sanitizer memcheck is closed on this pool): run with
LGM_WS_GUARD=1 so the library puts a 4 KiB guard band after every workspace region and every
n x n slot; every call below gets its guards filled before and checked after
(lgm_debug_ws_guard), and its device outputs sit between canary pads that are checked too.
Covers both engines (Engine F n = 32 / 48 / 64, G1 n = 80 / 100 / odd 101, G2 single-CTA
panels n = 320 / 512, G2 cluster panels n = 576), failure paths and every building block.

    LGM_WS_GUARD=1 python tools/guard_probe.py out.npz   -> one JSON line (per-call results)
Without LGM_WS_GUARD the same calls run unguarded (the test compares the two outputs bit for bit).
"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2401_10089_b200 import _lib, synth  # noqa: E402

P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
lib = _lib.load()
lib.lgm_debug_ws_guard.argtypes = [I64, I64, I32, P, I32, P, P]
lib.lgm_debug_ws_guard.restype = ctypes.c_int
dev = torch.device("cuda")
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
bad = torch.zeros(1, dtype=torch.int64, device=dev)
PAD = 2048
CANARY = np.uint64(0x7FF8DEADBEEF5A5A)
results, outputs = [], {}


def padded(nbytes):
    """device buffer of nbytes (8-byte aligned) between two canary pads of PAD words"""
    nw = (nbytes + 7) // 8
    buf = torch.from_numpy(np.full(nw + 2 * PAD, CANARY, dtype=np.uint64).view(np.int64)).to(dev)
    return buf, buf[PAD:PAD + nw], nw


def canary_ok(buf, nw):
    h = buf.cpu().numpy().view(np.uint64)
    return bool((h[:PAD] == CANARY).all() and (h[PAD + nw:] == CANARY).all())


def ws_for(n, b, block):
    nb = ctypes.c_size_t(0)
    (lib.lgm_block_workspace_bytes if block else lib.lgm_workspace_bytes)(n, b, ctypes.byref(nb))
    return torch.empty(max(int(nb.value), 8), dtype=torch.uint8, device=dev), int(nb.value)


def guarded(name, n, b, layout, ws, call, outs):
    """fill guards, call, check guards + output canaries; keep the outputs"""
    bad.zero_()
    filled = lib.lgm_debug_ws_guard(n, b, layout, ws.data_ptr(), 0, None, stream)
    rc = call()
    if filled:
        lib.lgm_debug_ws_guard(n, b, layout, ws.data_ptr(), 1, bad.data_ptr(), stream)
    torch.cuda.synchronize()
    ok = all(canary_ok(buf, nw) for buf, _, nw in outs)
    results.append({"call": name, "n": n, "batch": b, "rc": rc, "guarded": bool(filled), "bad": int(bad.item()),
                    "canary": ok})
    for i, (_, view, _) in enumerate(outs):
        outputs[f"{name}_{n}_{i}"] = view.cpu().numpy()


def dmat(A):
    return torch.from_numpy(np.ascontiguousarray(A)).to(dev)


def logm_case(cfg, n, b, A=None):
    A = dmat(synth.config(cfg, batch=b, n=n) if A is None else A)
    Lb, L, _ = padded(b * n * n * 8)
    Rb, R, _ = padded(b * 64)
    ws, nbytes = ws_for(n, b, False)
    o = _lib.Opts()
    lib.lgm_default_opts(ctypes.byref(o))
    call = lambda: lib.lgm_logm_f64(A.data_ptr(), L.data_ptr(), n, b, n, ctypes.byref(o), R.data_ptr(), ws.data_ptr(),
                                    nbytes, stream)
    guarded(f"logm{cfg}", n, b, 1 if n <= 64 else 0, ws, call, [(Lb, L, b * n * n), (Rb, R, b * 8)])


def blocks_case(n, b=2):
    A = synth.config("3b", batch=b, n=n)
    Ad = dmat(A)
    M = dmat(0.2 * (A - np.eye(n)) / np.abs(A - np.eye(n)).sum(axis=1).max(axis=1)[:, None, None])
    ws, nbytes = ws_for(n, b, True)
    w = (ws.data_ptr(), nbytes, stream)
    Xb, X, nx = padded(b * n * n * 8)
    ib, it, ni = padded(b * 4)
    sb, st, ns = padded(b * 4)
    guarded("sqrt_db", n, b, 0, ws, lambda: lib.lgm_sqrt_db_f64(Ad.data_ptr(), X.data_ptr(), n, b, n, 0.0, 50,
                                                               it.data_ptr(), st.data_ptr(), *w),
            [(Xb, X, nx), (ib, it, ni), (sb, st, ns)])
    eb, est, ne = padded(b * 8)
    pb, ps, npw = padded(b * 4)
    guarded("est_power", n, b, 0, ws, lambda: lib.lgm_est_power_norm_f64(M.data_ptr(), n, b, n, 3, 5, est.data_ptr(),
                                                                        ps.data_ptr(), *w), [(eb, est, ne), (pb, ps, npw)])
    guarded("est_product", n, b, 0, ws, lambda: lib.lgm_est_product_norm_f64(M.data_ptr(), 2, Ad.data_ptr(), n, b, n, 5,
                                                                            est.data_ptr(), ps.data_ptr(), *w),
            [(eb, est, ne), (pb, ps, npw)])
    Bb, Bm, nbm = padded(b * n * n * 8)
    cb, sc, nsc = padded(b * n * 8)
    guarded("balance", n, b, 0, ws, lambda: lib.lgm_balance_f64(Ad.data_ptr(), Bm.data_ptr(), sc.data_ptr(), n, b, n, 100,
                                                               st.data_ptr(), *w), [(Bb, Bm, nbm), (cb, sc, nsc), (sb, st, ns)])
    for k in (5, 7):
        guarded(f"degopt{k}", n, b, 0, ws, lambda: lib.lgm_eval_degopt_f64(M.data_ptr(), None, X.data_ptr(), n, b, n, k,
                                                                          it.data_ptr(), *w), [(Xb, X, nx), (ib, it, ni)])
    guarded("expm_ref", n, b, 0, ws, lambda: lib.lgm_expm_ref_f64(M.data_ptr(), X.data_ptr(), n, b, n, *w),
            [(Xb, X, nx)])


def selftest():
    """the checker sees a poked slot guard byte and a poked region-tail byte (guarded runs only)"""
    n, b = 80, 2
    ws, nbytes = ws_for(n, b, True)
    bad.zero_()
    if not lib.lgm_debug_ws_guard(n, b, 0, ws.data_ptr(), 0, None, stream):
        return None
    ws[n * n * 8 + 5] = 0                    # guard band after slot (0, 0)
    ws[nbytes - 1] = 0                       # guard band after the last region
    lib.lgm_debug_ws_guard(n, b, 0, ws.data_ptr(), 1, bad.data_ptr(), stream)
    fw, fb = ws_for(32, 2, False)
    lib.lgm_debug_ws_guard(32, 2, 1, fw.data_ptr(), 0, None, stream)
    fw[(8 * 32 * 32) * 8] = 0                # Engine F: guard band after matrix 0's workspace
    lib.lgm_debug_ws_guard(32, 2, 1, fw.data_ptr(), 1, bad.data_ptr(), stream)
    torch.cuda.synchronize()
    return int(bad.item())


def main():
    detected = selftest()
    for cfg, n, b in ((2, 32, 3), ("3b", 48, 2), (1, 64, 1), ("3b", 80, 2), ("3b", 100, 2), (2, 101, 2), (4, 320, 2),
                      (4, 512, 2), ("5b", 576, 1)):
        logm_case(cfg, n, b)
    # failure paths: non-finite, negative eigenvalue (DB non-convergence), exactly singular
    for n in (40, 80):
        A = np.stack([np.full((n, n), np.nan), np.diag(np.r_[-1.0, np.linspace(2, 3, n - 1)]),
                      np.diag(np.r_[0.0, np.linspace(2, 3, n - 1)])])
        logm_case("fail", n, 3, A)
    for n in (48, 80, 320):
        blocks_case(n)
    np.savez(sys.argv[1] if len(sys.argv) > 1 else "/tmp/guard_probe.npz", **outputs)
    print(json.dumps({"selftest_detected": detected, "calls": results}))


if __name__ == "__main__":
    main()
