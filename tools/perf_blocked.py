"""Time blocked BO sweeps on config 3 (exploration).

SWEEPS=n (default 1), NBLK=list (default 128), TUNE="nsplit,..." (Gram row splits,
ghsvd_options.gram_splits; default: planned)."""
import json
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_08560_b200 import build, ghsvd, inputs  # noqa: E402

build.build()
warnings.simplefilter("ignore")
kind, at = inputs.make_config(3, backend="torch")
NA, NL, NG = at.A.shape
sweeps = int(os.environ.get("SWEEPS", "1"))
tunes = [t for t in os.environ.get("TUNE", "").split(",") if t] or [None]
for nb in [int(x) for x in os.environ.get("NBLK", "128").split(",")]:
    for tune in tunes:
        ctx = ghsvd.Context(2 * NA * NL, NG, NL, variant="bo", nblocks=nb, max_sweeps=sweeps, detail_timing=True,
                            gram_splits=int(tune) if tune else None)
        ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
        st = ctx.sweep()
        print(json.dumps({"nblk": nb, "tune": tune, "sweeps": st["sweeps"], "converged": st["converged"],
                          "kernel_s": st["kernel_seconds"], "s_per_sweep": st["kernel_seconds"] / st["sweeps"],
                          "TFLOPs": st["alg_flops"] / st["kernel_seconds"] / 1e12,
                          "t_gram": st["t_gram"], "t_pivot": st["t_pivot"], "t_update": st["t_update"],
                          "big": st["big_per_sweep"][-3:]}), flush=True)
        ctx.close()
