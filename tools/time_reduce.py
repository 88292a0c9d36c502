"""Time ghsvd_reduce (Phase 2) on a BASELINE config, blocked vs unblocked, plain vs
column-pivoted, and check that each preserves the Grammians (eq 5.1):
P^T F~^* J~ F~ P = F^* J F and likewise for G (products by torch on the GPU: checking only).

  python tools/time_reduce.py [--config 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--modes", nargs="*", default=["blocked", "unblocked", "blocked_colpiv", "unblocked_colpiv"])
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1907_08560_b200 import build, ghsvd, inputs
    build.build()
    kind, at = inputs.make_config(args.config, backend="torch")
    NA, NL, NG = at.A.shape
    m, n = 2 * NA * NL, NG
    dev = "cuda"
    for mode in args.modes:
        ctx = ghsvd.Context(m, n, NL, variant="bo")
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        o = n & 1   # odd n: the factors are exported bordered (one more row and column)
        Ft = torch.empty((n + o, m + o), dtype=torch.complex128, device=dev).t()
        Gt = torch.empty((n + o, m + o), dtype=torch.complex128, device=dev).t()
        Jt = torch.empty(m + o, dtype=torch.int8, device=dev)
        ctx.export_factors(Ft, Jt, Gt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.reduce(colpiv="colpiv" in mode, unblocked=mode.startswith("unblocked"), colsearch="colsearch" in mode)
        e1.record()
        torch.cuda.synchronize()
        secs = e0.elapsed_time(e1) * 1e-3
        Fr = torch.empty((n + o, n + o), dtype=torch.complex128, device=dev).t()
        Gr = torch.empty((n + o, n + o), dtype=torch.complex128, device=dev).t()
        Jr = torch.empty(n + o, dtype=torch.int8, device=dev)
        ctx.export_factors(Fr, Jr, Gr)
        _, _, _, p2 = ctx.get_factors() if n <= 2048 else (None, None, None, None)
        if p2 is None:   # p2 only (avoid copying the factors to the host)
            import ctypes
            p2 = np.zeros(n, np.int64)
            mm, nn = ctypes.c_int64(), ctypes.c_int64()
            ctx._L.ghsvd_get_factors(ctx._h, ctypes.byref(mm), ctypes.byref(nn), None, 0, None, None, 0,
                                     p2.ctypes.data_as(ctypes.c_void_p))
        pt = torch.from_numpy(p2).to(dev)
        H = (Ft.conj().T @ (Jt.double()[:, None] * Ft))[:n, :n]
        S = (Gt.conj().T @ Gt)[:n, :n]
        Hr = (Fr.conj().T @ (Jr.double()[:, None] * Fr))[:n, :n]
        Sr = (Gr.conj().T @ Gr)[:n, :n]
        eh = float(torch.linalg.norm(Hr - H[pt][:, pt]) / torch.linalg.norm(H))
        es = float(torch.linalg.norm(Sr - S[pt][:, pt]) / torch.linalg.norm(S))
        print(json.dumps({"config": args.config, "mode": mode, "seconds": secs,
                          "fallback_col": getattr(ctx, "reduce_fallback_col", None), "grammian_err_H": eh,
                          "grammian_err_S": es, "m": m, "n": n}), flush=True)
        ctx.close()
        del Ft, Gt, Fr, Gr, H, S, Hr, Sr
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
