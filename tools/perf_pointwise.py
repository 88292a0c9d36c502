"""Exploration: time one pointwise sweep of config 3 for several launch configurations,
and measure cuBLAS FP64 / complex128 GEMM peaks (roofline denominators for the blocked path)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1907_08560_b200 import build, ghsvd, inputs

build.build()
out = {}
if "--peaks" in sys.argv:
    for dt, name in ((torch.float64, "dgemm"), (torch.complex128, "zgemm")):
        n = 8192 if dt == torch.float64 else 4096
        a = torch.randn(n, n, dtype=dt, device="cuda"); b = torch.randn(n, n, dtype=dt, device="cuda")
        for _ in range(2): a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
        fl = 2 * n ** 3 * (4 if dt == torch.complex128 else 1)
        out[name + "_tflops"] = fl / best / 1e9
    print(json.dumps(out), flush=True)
kind, at = inputs.make_config(3, backend="torch")
NA, NL, NG = at.A.shape
m, n = 2 * NA * NL, NG
cfgs = [(8, 256, 2), (8, 128, 2), (4, 256, 2), (16, 256, 2), (8, 512, 2), (4, 512, 2), (8, 256, 1)]
for arg in sys.argv[1:]:
    if arg.startswith("--cfg="):
        cfgs = [tuple(int(x) for x in c.split("x")) for c in arg[6:].split(",")]
for C, T, K in cfgs:
    ctx = ghsvd.Context(m, n, NL, cluster=C, threads=T, max_sweeps=1, kernel=K)
    ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
    import warnings; warnings.simplefilter("ignore")
    st = ctx.sweep()
    gbs = st["alg_bytes"] / st["kernel_seconds"] / 1e9
    print(json.dumps({"C": C, "T": T, "K": K, "sweep_s": st["kernel_seconds"], "GBs": gbs,
                      "us_per_launch": st["kernel_seconds"] / st["launches"] * 1e6}), flush=True)
    ctx.close()
