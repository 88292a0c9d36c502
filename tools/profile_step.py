"""Run a few steps on config 3 (for ncu captures of k_pair_step / the k_blk_* kernels).
usage: python tools/profile_step.py [--variant pointwise|bo] [--kernel K] [--cluster C]
       [--threads T] [--steps S] [--sweep]
A pointwise step is one k_pair_step launch.  Blocked (bo): --steps runs block steps
through the single-stream diagnostic ghsvd_run_steps (1 Gram + 1 pivot + 1 update
launch per step over all block pairs); --sweep instead runs ONE full block sweep with
the bench's schedule (per block step: Gram, pivot and F/G-update launches for each half
of the pairs, then the Z' update), i.e. the exact launches bench.py times."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1907_08560_b200 import build, ghsvd, inputs
ap = argparse.ArgumentParser()
ap.add_argument("--kernel", type=int, default=1)
ap.add_argument("--cluster", type=int, default=0)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--variant", default="pointwise")
ap.add_argument("--sweep", action="store_true")
a = ap.parse_args()
build.build()
kind, at = inputs.make_config(3, backend="torch")
NA, NL, NG = at.A.shape
if a.variant == "pointwise":
    ctx = ghsvd.Context(2 * NA * NL, NG, NL, kernel=a.kernel, cluster=a.cluster, threads=a.threads,
                        max_sweeps=1)
else:
    ctx = ghsvd.Context(2 * NA * NL, NG, NL, variant=a.variant, max_sweeps=1)
ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(torch.cuda.current_stream())
if a.sweep:
    st = ctx.sweep()
    e1.record(torch.cuda.current_stream()); torch.cuda.synchronize()
    print("one sweep", st["seconds"], "s")
else:
    ctx.run_steps(0, a.steps)
    e1.record(torch.cuda.current_stream()); torch.cuda.synchronize()
    print("steps", a.steps, "ms/step", e0.elapsed_time(e1) / a.steps)
