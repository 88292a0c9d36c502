#!/usr/bin/env python
"""Benchmark of the GHSVD sweep engine (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3] [--variant pointwise|bo] [--cluster C] [--threads T]

One "step" = one complete Phase-3 solve (ghsvd_sweep to convergence: all sweeps of
the round-robin HZ iteration) on BASELINE configs[3]
(N_A=64, N_L=81, N_G=4096: F, G 10368 x 4096 complex128, ill-conditioned S, J 50 %
negative), from the factors Phase 1 (ghsvd_factor, timed separately) produced.

* value  = time-to-converge in seconds, device time (CUDA events on the context
           stream) of ghsvd_sweep with the factors already resident in HBM; mean of
           the K timed steps, max over ranks.  Inputs (1.6 GB) exceed L2 (126 MB).
* e2e    = the same solve through the C ABI from pinned HOST buffers: H2D of F, G, J
           (ghsvd_set_factors) + sweep + D2H of lambda, Sigma_F, Sigma_G (ghsvd_extract).
* roofline: blocked (default): the dominant kernel k_blk_update (F, G row tiles);
           algorithmic flops 8 k^2 (2m) per block pair (k = block-pivot order) / its
           summed CUDA-event time; peak = cuBLAS ZGEMM measured live.  Pointwise:
           k_pair_step_2p, algorithmic bytes (128m+64n per transformed pair, 64m per
           skipped pair, from the device counters) / time; peak = MEASURED_PEAKS hbm_gbs.
* cpu_baseline: the oracle (oracle/, plain C + OpenMP) timed on a bounded sample
           (a few steps of sweep 1 on the same factors), extrapolated to the GPU's
           sweep count.
"""
from __future__ import annotations

import argparse
import json
import os
import warnings
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GHSVD time-to-converge (s) c128 N_G=4096"
UNIT = "s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_factors(cfg: int, backend: str):
    from paper_1907_08560_b200 import inputs
    return inputs.make_config(cfg, backend=backend)


def launch_cmd(nproc: int, argv, port: int):
    """The torchrun command bench.py re-executes itself under for --gpus N > 1 when it was
    not started by torchrun (one process per GPU, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shared_inputs(cfg: int, ws: int, rank: int, dev):
    """Seeded inputs generated ONCE (rank 0, host numpy: the stored oracle references were
    computed on exactly these atoms) and broadcast to the other ranks over NCCL, so every
    rank factors bitwise-identical atoms."""
    import torch
    if ws == 1:
        return make_factors(cfg, "numpy")
    import torch.distributed as dist
    from paper_1907_08560_b200 import inputs
    obj = [None]
    if rank == 0:
        kind, payload = make_factors(cfg, "numpy")
        names = ["A", "B", "U", "TAA", "TAB", "TBB", "d"] if kind == "atoms" else ["F", "J", "G"]
        arrs = {k: np.ascontiguousarray(getattr(payload, k)) for k in names}
        obj = [(kind, {k: (a.shape, str(a.dtype)) for k, a in arrs.items()},
                None if kind == "atoms" else payload.lam_true)]
    dist.broadcast_object_list(obj, 0)
    kind, meta, lam_true = obj[0]
    out = {}
    for k, (shp, dt) in meta.items():
        nbytes = int(np.prod(shp)) * np.dtype(dt).itemsize
        host = arrs[k].view(np.uint8).reshape(-1) if rank == 0 else np.zeros(nbytes, np.uint8)
        t = torch.from_numpy(host).to(dev)
        dist.broadcast(t, 0)
        out[k] = t.cpu().numpy().view(np.dtype(dt)).reshape(shp)
    if kind == "atoms":
        return kind, inputs.Atoms(**out)
    return kind, inputs.Pencil(out["F"], out["J"], out["G"], lam_true=lam_true)


def stored_oracle_parity(cfg: int, at, lam, phase2=None):
    """Max relative eigenvalue error of this run against the stored oracle reference for
    the config, written by the oracle-only script tools/make_oracle_reference.py from the
    same seeded atoms: tests/golden/c<cfg>_oracle_pointwise (HZ, Alg. 2; config 3, north-star
    tolerance 1e-6; config 5, 1e-9) or c<cfg>_oracle_dense (H and S formed, ZHEGVD,
    PAPER.md:818-836; configs 4 and 6, well-conditioned S, tolerance 1e-9); None if there is
    none.  `at` is the config's seeded atoms or pencil (keyed by inputs.fingerprint)."""
    from paper_1907_08560_b200 import inputs
    gold = os.path.join(ROOT, "tests", "golden")
    # north-star tolerances: 1e-6 on the ill-conditioned config 3, 1e-9 elsewhere; 1e-8
    # through Phase 2 against an unreduced reference (reading R2-3)
    through_p2 = bool(phase2) or "reduce" in inputs.CONFIGS[cfg].get("entry", "")
    stem, tol = os.path.join(gold, f"c{cfg}_oracle_pointwise"), 1e-6 if cfg == 3 else 1e-9
    if not os.path.exists(stem + ".json"):
        stem, tol = os.path.join(gold, f"c{cfg}_oracle_dense"), 1e-9
        if not os.path.exists(stem + ".json"):
            return None
    if through_p2 and cfg != 3:
        tol = 1e-8
    meta = json.load(open(stem + ".json"))
    ok = inputs.fingerprint_close(inputs.fingerprint(at), meta["fingerprint"])
    lo = np.sort(np.load(stem + ".npz")["lam"])
    la = np.sort(np.asarray(lam))
    err = float(np.max(np.abs(la - lo) / np.abs(lo))) if ok and la.shape == lo.shape else None
    out = {"reference": os.path.relpath(stem, ROOT) + ".{json,npz}", "inputs_match": bool(ok),
           "max_rel_lambda_err": err, "tol": tol, "within_tol": err is not None and err <= tol,
           "oracle_sweeps": meta["stats"]["sweeps"],
           "oracle_seconds_measured": meta.get("seconds_sweep", meta.get("seconds_solve")),
           "oracle_threads": meta["threads"], "oracle_cpu": meta["cpu_model"]}
    if phase2:
        out["note"] = ("Phase 2 (QR of the badly conditioned G) costs accuracy on this pencil, as "
                       "PAPER.md:925-927 warns; the metric's recipe skips it (DESIGN.md Sec 8)")
    return out


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def oracle_factors(kind, payload, cfg: int):
    """The sweep's starting factors computed by the ORACLE from the seeded inputs (its own
    Phase 1, and Phase 2 where the config's recipe has it): nothing from the CUDA path."""
    import oracle
    from paper_1907_08560_b200 import inputs
    if kind == "atoms":
        F, J, G = oracle.factor(payload.A, payload.B, payload.U, payload.TAA, payload.TAB, payload.TBB)
        if "reduce" in inputs.CONFIGS[cfg].get("entry", ""):
            F, J, G, _, _ = oracle.reduce(F, J, G)
        return F, J, G
    return payload.F, payload.J, payload.G


def _stored_stats(cfg: int):
    """Sweep count and per-sweep transformation counts of the stored oracle solve of this
    config (tests/golden/c<cfg>_oracle_pointwise.json, oracle-only), if any."""
    p = os.path.join(ROOT, "tests", "golden", f"c{cfg}_oracle_pointwise.json")
    if not os.path.exists(p):
        return None
    m = json.load(open(p))
    return {"sweeps": m["stats"]["sweeps"], "all_per_sweep": m["stats"]["all_per_sweep"],
            "seconds_measured": m["seconds_sweep"], "threads": m["threads"], "cpu_model": m["cpu_model"],
            "file": os.path.relpath(p, ROOT)}


def cpu_baseline_sample(F0, J0, G0, cfg: int, fallback_sweeps: int, budget_s: float = 15.0):
    """The oracle (as it stands) on the host cores, Algorithm 2 pointwise.

    Small problems (a whole solve fits the budget) are timed END TO END.  Otherwise a
    bounded sample is timed and extrapolated with a two-term cost model of a round-robin
    step: every pair pays a Gram pass (c_g per pair), transformed pairs also their
    updates (c_u).  c_g + c_u comes from steps of sweep 1 on the real factors (every pair
    is transformed there), c_g from the same steps on [I; 0] factors (h_pq = s_pq = 0:
    nothing is transformed, same m, n, same memory traffic).  The sweep count and the
    per-sweep transformation counts are the ORACLE's own, from its stored full solve of
    this config (tests/golden); without one, every pair of `fallback_sweeps` sweeps is
    counted as transformed (an upper bound), and the line says so."""
    import oracle
    m, n = F0.shape
    cores = _cores()
    base = {"unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model()}
    Z = np.eye(n, dtype=np.complex128, order="F")
    # whole solve if it fits the budget (a sweep costs at most n-1 all-transformed steps)
    t = time.perf_counter()
    oracle.hz_steps(F0, J0, G0, Z, 0, min(n - 1, 8))
    t_est = (time.perf_counter() - t) / min(n - 1, 8) * (n - 1) * max(fallback_sweeps, 1)
    if t_est <= budget_s:
        t = time.perf_counter()
        _, _, _, st = oracle.hz_pointwise(F0, J0, G0, cmax=64, nthreads=cores)
        tt = time.perf_counter() - t
        return dict(base, value=tt, sample=f"whole oracle solve timed end to end ({st['sweeps']} sweeps, "
                                             f"{m}x{n}, pointwise Alg. 2)", measured=True, sweeps=st["sweeps"])
    E = np.zeros((m, n), dtype=np.complex128, order="F")
    E[np.arange(n), np.arange(n)] = 1.0
    JE = np.ones(m, dtype=np.int8)

    def per_step(F, J, G, budget):
        # each call copies F, G, Z first: per-step cost = (t(1 + ns) - t(1)) / ns, after one
        # untimed call (first-touch page faults of the copies inflate the first call).  ns
        # doubles until the steps alone take half the budget or the calls the whole budget:
        # the time stays bounded even when the copy overhead swamps a short probe (a probe
        # of 4 Gram-only steps once extrapolated to a 33 s sample)
        oracle.hz_steps(F, J, G, Z, 0, 1)
        t = time.perf_counter()
        oracle.hz_steps(F, J, G, Z, 0, 1)
        ta = time.perf_counter() - t
        ns, total = 4, ta
        while True:
            t = time.perf_counter()
            oracle.hz_steps(F, J, G, Z, 0, 1 + ns)
            tc = time.perf_counter() - t
            total += tc
            if tc - ta >= 0.5 * budget or total >= budget or ns >= n - 2:
                break
            ns = min(n - 2, 2 * ns)
        return max(tc - ta, 1e-9) / ns, ns, total

    c_full, ns_f, s1 = per_step(F0, J0, G0, 0.7 * budget_s)
    c_gram, ns_g, s2 = per_step(E, JE, E, 0.3 * budget_s)
    pairs_step = n // 2
    cg, cu = c_gram / pairs_step, max(c_full - c_gram, 0.0) / pairs_step
    ref = _stored_stats(cfg)
    if ref is not None:
        sweeps, allp = ref["sweeps"], ref["all_per_sweep"]
        how = f"the oracle's own {sweeps} sweeps and per-sweep transformation counts ({ref['file']})"
    else:
        sweeps, allp = fallback_sweeps, [n * (n - 1) // 2] * fallback_sweeps
        how = f"{sweeps} sweeps with every pair transformed (no stored oracle solve of this config: upper bound)"
    value = sum((n - 1) * pairs_step * cg + a * cu for a in allp)
    out = dict(base, value=value, measured=False, sweeps=sweeps,
               sample=(f"steps 1..{ns_f} of sweep 1 on the oracle's own {m}x{n} starting factors "
                       f"({c_full:.4f} s/step, all pairs transformed) and steps 1..{ns_g} on [I;0] factors "
                       f"({c_gram:.4f} s/step, Gram passes only), extrapolated with {how}"),
               seconds_measured=s1 + s2, c_gram_per_pair=cg, c_update_per_pair=cu)
    if ref is not None:
        out["stored_full_solve"] = {"seconds": ref["seconds_measured"], "threads": ref["threads"],
                                    "cpu_model": ref["cpu_model"], "measured": True}
    return out


# sweeps the GPU (BO) solve of each config takes: fallback of the extrapolation when no
# stored oracle solve exists for the config
REF_SWEEPS = {0: 7, 1: 18, 2: 13, 3: 36, 4: 14, 5: 17, 6: 14}


def cpu_baseline_fresh_process(cfg: int, sweeps: int, budget_s: float):
    """cpu_baseline_sample in a FRESH process (this script's --impl reference leg, one
    step): in the bench process, beside its CUDA context and torch's threads, the oracle's
    OpenMP update passes measured ~1.6x slower per pair than in the reference arm's own
    process on the same host, so the two lines disagreed by tens of percent.  Returns
    (cpu_baseline, None), or (None, error) if the child fails (the caller then samples
    in-process and says so)."""
    drop = ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "GROUP_RANK", "ROLE_RANK", "MASTER_ADDR",
            "MASTER_PORT", "TORCHELASTIC_RUN_ID")
    env = {k: v for k, v in os.environ.items() if k not in drop}
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--config", str(cfg), "--steps", "1",
           "--warmup", "0", "--ref-budget", str(budget_s), "--ref-sweeps", str(max(sweeps, 1))]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
        js = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode == 0 and js:
            cb = json.loads(js[-1])["cpu_baseline"]
            cb["process"] = "fresh process (bench.py --impl reference --steps 1 --warmup 0)"
            return cb, None
        err = (r.stderr or "")[-300:]
    except (subprocess.SubprocessError, OSError, ValueError, KeyError) as e:
        err = repr(e)
    return None, err


def run_reference(args):
    """--impl reference: the oracle as it stands, on host cores, same config/metric."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_1907_08560_b200 import inputs
    kind, payload = make_factors(args.config, "numpy")
    F0, J0, G0 = oracle_factors(kind, payload, args.config)
    sweeps = args.ref_sweeps if args.ref_sweeps > 0 else REF_SWEEPS.get(args.config, 36)
    m, n = F0.shape
    vals = []
    # each step is a bounded sample; the whole --steps K --warmup W run stays within a few
    # minutes (about 8 x ref_budget of sampling in total once K + W exceeds 8)
    per_step = args.ref_budget if args.warmup + args.steps <= 8 else \
        max(2.0, 8.0 * args.ref_budget / (args.warmup + args.steps))
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline_sample(F0, J0, G0, args.config, sweeps, budget_s=per_step)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = float(np.mean(vals))
    cb["value"] = v
    line = {"impl": "reference", "metric": metric_name(args.config, n), "value": v, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": inputs.CONFIGS[args.config]["name"], "m": m, "n": n,
                       "variant": "oracle-pointwise", "sweeps_extrapolated": None if cb["measured"] else cb["sweeps"],
                       "phase2": "oracle.reduce" if "reduce" in inputs.CONFIGS[args.config].get("entry", "")
                       else "none"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfg: int, n: int) -> str:
    return METRIC if cfg == 3 else f"GHSVD time-to-converge (s) c128 N_G={n} (config {cfg})"


def measure_zgemm_peak(dev) -> float:
    """Live FP64 tensor-core roofline denominator: cuBLAS ZGEMM (complex128) TFLOP/s,
    best of 10 at 4096^3 (MEASURED_PEAKS.json has no FP64 figure); nvidia-smi clocks are
    sampled around it (roofline.peak_clocks)."""
    import torch
    a = torch.randn(4096, 4096, dtype=torch.complex128, device=dev)
    b = torch.randn(4096, 4096, dtype=torch.complex128, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize(dev)
    best = 1e30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b
    return 8.0 * 4096 ** 3 / best / 1e12


def _ncu_traffic(kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu summary, if any."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        k = d.get("kernels", {}).get(kernel)
        return None if k is None else k.get("dram_bytes_per_launch")
    except Exception:
        return None


def run_ours(args):
    import torch
    from paper_1907_08560_b200 import build, ghsvd, inputs
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        if args.variant == "pointwise":
            args.variant = "bo"                     # only the blocked variant shards
    build.build()
    stream = torch.cuda.Stream(dev)
    cfg = inputs.CONFIGS[args.config]
    blocked = args.variant in ("bo", "fb")
    zgemm_peak, zgemm_clocks = None, None
    if blocked:
        with ClockSampler(local) as zclk:
            zgemm_peak = measure_zgemm_peak(dev)
        zgemm_clocks = zclk.summary()
    # ---- inputs (seeded, synthetic; generated once and broadcast) and Phase 1 on the device
    kind, payload = shared_inputs(args.config, ws, rank, dev)
    if kind == "atoms":
        at = payload
        NA, NL, NG = at.A.shape
        m, n, nl = 2 * NA * NL, NG, NL
    else:
        m, n = payload.F.shape
        nl = 0
    nccl_id = None
    if ws > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(ghsvd.nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    # block ordering (blocked variants; DESIGN.md 6 "Level-3 orderings", reading R2-5): HIER by
    # default -- each block pair once per sweep grouped by super pair, 2P - 1 exchanges per
    # sweep on P GPUs; --ordering rr is the paper's round-robin (reading C-11)
    ordering = args.ordering if blocked else "rr"
    ctx = ghsvd.Context(m, n, nl, variant=args.variant, device=local, stream=stream, max_sweeps=args.max_sweeps,
                        cluster=args.cluster, threads=args.threads, nblocks=args.nblocks, world_size=ws,
                        rank=rank, nccl_id=nccl_id, detail_timing=2 if blocked else 0, want_x=args.want_x,
                        ordering=ordering, super_blocks=args.super_blocks)
    phase1_s = None
    phase2_s = None
    with torch.cuda.stream(stream):
        if kind == "atoms":
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(stream)
            ctx.factor(at.A, at.B, at.U, at.TAA, at.TAB, at.TBB)
            ev[1].record(stream)
            stream.synchronize()
            phase1_s = ev[0].elapsed_time(ev[1]) * 1e-3
            if "reduce" in cfg.get("entry", "") or args.reduce == "colpiv":
                t0 = time.perf_counter()
                # Phase 2: config 2 recipe, or (--reduce colpiv) the column-pivoted QR of
                # G P2 that PAPER.md:925-943 gives for a badly conditioned G~
                ctx.reduce(colpiv=args.reduce == "colpiv")
                torch.cuda.synchronize(dev)
                phase2_s = time.perf_counter() - t0
        else:
            ctx.set_factors(payload.F, payload.J, payload.G)
        mb, nb = ctx.factor_shape()
        # pinned host copies of the starting factors: the e2e inputs of every step
        Fh = torch.empty((nb, mb), dtype=torch.complex128, pin_memory=True).t()
        Gh = torch.empty((nb, mb), dtype=torch.complex128, pin_memory=True).t()
        Jh = torch.empty(mb, dtype=torch.int8, pin_memory=True)
        ctx.export_factors(Fh, Jh, Gh)
        stream.synchronize()
        if nb != n:
            # odd n: the exported factors carry the sweep's border row / column (last, C-10);
            # the e2e input is the unbordered problem (set_factors borders it again)
            mb, nb = mb - 1, nb - 1
            Fh, Gh, Jh = Fh[:mb, :nb], Gh[:mb, :nb], Jh[:mb]
    identical = None
    if ws > 1:
        # every rank must start from bitwise the same factors (deterministic Phase 1 on
        # identical atoms): compare digests of the exported factors
        import hashlib
        import torch.distributed as dist
        hs = hashlib.sha256()
        for t in (Fh, Gh, Jh):
            hs.update(t.contiguous().numpy().tobytes() if t.is_contiguous() else t.t().contiguous().numpy().tobytes())
        dig = [None] * ws
        dist.all_gather_object(dig, hs.hexdigest())
        identical = len(set(dig)) == 1
        if not identical:
            raise SystemExit(f"rank {rank}: starting factors differ across ranks ({dig})")
    lam_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    sf_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    sg_h = torch.empty(n, dtype=torch.float64, pin_memory=True)

    def one_step():
        """e2e: H2D of F, J, G (pinned) -> Phase 3 to convergence -> D2H of lambda, Sigma_F, Sigma_G.
        value: the sweep alone (factors resident in HBM)."""
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(stream):
            e[0].record(stream)
            ctx.set_factors(Fh, Jh, Gh)
            e[1].record(stream)
            st = ctx.sweep()
            e[2].record(stream)
            ctx.extract(want_z=False, out=(lam_h, sf_h, sg_h, None))
            e[3].record(stream)
        stream.synchronize()
        return st, e[1].elapsed_time(e[2]) * 1e-3, e[0].elapsed_time(e[3]) * 1e-3

    for _ in range(args.warmup):
        one_step()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    dev_t, e2e_t, stats = [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            st, td, te = one_step()
            dev_t.append(td)
            e2e_t.append(te)
            stats.append(st)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    value = float(np.mean(dev_t))
    e2e = float(np.mean(e2e_t))
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([value, e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        value, e2e = float(t[0]), float(t[1])
    launches = sum(s["launches"] for s in stats)
    sweeps = stats[-1]["sweeps"]
    pairs = stats[-1]["pairs_visited"]
    peaks = _peaks()
    if blocked:
        # dominant kernel: k_blk_update over the F and G row tiles; "achieved" uses its
        # CUDA-event spans on its launching stream over the timed region.  In the timed
        # schedule the two halves' kernels overlap (that is the point of the schedule), so
        # a span also contains other kernels' work: the value is a lower bound.  The
        # "isolated" entry times the same kernels live in this run on a one-sweep probe
        # with GHSVD_SERIAL=1 (every kernel alone on the stream, one launch per kind and
        # step), and "whole_step_tflops" is all algorithmic flops / the timed sweep time.
        t_upd = sum(s["t_update_fg"] for s in stats)
        f_upd = sum(s["flops_update_fg"] for s in stats)
        n_upd = sum(s["launches_update_fg"] for s in stats)
        iso = None
        if ws == 1:
            cp = ghsvd.Context(m, n, nl, variant=args.variant, device=local, stream=stream, max_sweeps=1,
                               nblocks=args.nblocks, detail_timing=True, schedule=ghsvd.SCHED_SERIAL,
                               ordering=ordering, super_blocks=args.super_blocks)
            with torch.cuda.stream(stream), warnings.catch_warnings():
                warnings.simplefilter("ignore")   # one-sweep probe: "not converged" is expected
                cp.set_factors(Fh, Jh, Gh)
                sp = cp.sweep()
            stream.synchronize()
            cp.close()
            ia = sp["flops_update_fg"] / sp["t_update_fg"] / 1e12 if sp["t_update_fg"] > 0 else 0.0
            ig = sp["flops_gram"] / sp["t_gram"] / 1e12 if sp["t_gram"] > 0 else 0.0
            iso = {"achieved": ia, "frac": ia / zgemm_peak, "launches": int(sp["launches_update_fg"]),
                   "alg_flops_per_launch": sp["flops_update_fg"] / max(sp["launches_update_fg"], 1),
                   "avg_launch_us": sp["t_update_fg"] / max(sp["launches_update_fg"], 1) * 1e6,
                   "k_blk_gram_achieved": ig, "k_blk_gram_frac": ig / zgemm_peak,
                   "k_blk_gram_note": "span includes the fused HEBPJ / Cholesky tail of the last pairs",
                   "probe": "1 sweep, schedule SERIAL, same factors, CUDA events on the context stream"}
        t_gr = sum(s["t_gram"] for s in stats)
        f_gr = sum(s["flops_gram"] for s in stats)
        t_pv = sum(s["t_pivot"] for s in stats)
        ach = f_upd / t_upd / 1e12 if t_upd > 0 else 0.0
        if t_gr > 0:   # full detail timing in the timed region
            others = {"k_blk_gram": {"achieved": f_gr / t_gr / 1e12, "frac": (f_gr / t_gr / 1e12) / zgemm_peak,
                                     "seconds": t_gr,
                                     "note": "event span includes the fused HEBPJ / pivoted-Cholesky tail "
                                             "and the concurrent Grams of the other half"},
                      "k_blk_pivot": {"seconds": t_pv, "bound": "latency (inner one-sided sweep in shared memory)"}}
        elif iso is not None:   # the timed region records only the update spans (detail_timing 2)
            others = {"k_blk_gram": {"achieved": iso["k_blk_gram_achieved"], "frac": iso["k_blk_gram_frac"],
                                     "seconds_per_sweep": sp["t_gram"],
                                     "note": "isolated probe (schedule SERIAL, one sweep); span includes the fused "
                                             "HEBPJ / pivoted-Cholesky tail"},
                      "k_blk_pivot": {"seconds_per_sweep": sp["t_pivot"], "note": "isolated probe",
                                      "bound": "latency (inner one-sided sweep in shared memory)"}}
        else:
            others = None
        roof = {"bound": "tensor", "achieved": ach, "peak": zgemm_peak, "unit": "TFLOP/s",
                "frac": ach / zgemm_peak, "traffic": _ncu_traffic("k_blk_update"), "kernel": "k_blk_update",
                "alg_flops_per_launch": f_upd / max(n_upd, 1), "avg_launch_us": t_upd / max(n_upd, 1) * 1e6,
                "launches": int(n_upd),
                "flops_unit": "8 real flops per complex multiply-add (4M-equivalent; the kernel runs the 3M "
                              "scheme, so it can exceed the 4M ZGEMM rate)",
                "peak_clocks": zgemm_clocks,
                "peak_source": "cuBLAS ZGEMM 4096^3 measured live in this run (FP64 DMMA; MEASURED_PEAKS.json "
                               "has no FP64 figure)",
                "others": others,
                "isolated": iso,
                "whole_step_tflops": sum(s["alg_flops"] for s in stats) / sum(s["kernel_seconds"] for s in stats) / 1e12}
        roof["whole_step_frac"] = roof["whole_step_tflops"] / zgemm_peak
    else:
        kern_s = sum(s["kernel_seconds"] for s in stats)
        alg = sum(s["alg_bytes"] for s in stats)
        peak = peaks.get("hbm_gbs", 6650.0)
        achieved = alg / kern_s / 1e9 if kern_s > 0 else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": _ncu_traffic("k_pair_step_2p"), "kernel": "k_pair_step_2p",
                "alg_bytes_per_launch": alg / max(launches, 1), "avg_launch_us": kern_s / max(launches, 1) * 1e6,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"}
    if rank != 0:
        ctx.close()
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0
    metric = metric_name(args.config, n)
    line = {
        "metric": metric, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": cfg["name"], "m": mb, "n": nb, "variant": args.variant, "max_sweeps": args.max_sweeps,
                   "ordering": ordering if blocked else "round-robin (pointwise)",
                   "nblocks": stats[-1].get("nblocks") if blocked else None,
                   "super_blocks": stats[-1].get("super_blocks") if blocked and ordering != "rr" else None,
                   "want_x": bool(args.want_x),
                   "l2": f"inputs ({2 * mb * nb * 16 / 1e9:.2f} GB) vs L2 126 MB",
                   "phase2": ("column-pivoted QR of G P2 (--reduce colpiv, PAPER.md:925-943)" if args.reduce == "colpiv"
                              else "applied" if phase2_s is not None
                              else "skipped (config recipe; PAPER.md:925 for ill-conditioned G)")},
        "sweeps": sweeps, "converged": stats[-1]["converged"], "big_per_sweep_tail": stats[-1]["big_per_sweep"][-4:],
        "max_offdiag_last_sweep": stats[-1]["max_offdiag_last"],
        "seconds_per_sweep": value / max(sweeps, 1),
        "pair_updates_per_s": pairs / value, "transforms_per_s": stats[-1]["transforms_all"] / value,
        "phase1_seconds": phase1_s, "phase2_seconds": phase2_s,
        "roofline": roof,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(2 * mb * nb * 16 + mb),
                "d2h_bytes_per_step": int(3 * n * 8)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if identical is not None:
        line["inputs_identical_across_ranks"] = identical
    # every config with a stored oracle reference (atoms or a pencil)
    par = stored_oracle_parity(args.config, payload, lam_h.numpy(), phase2=args.reduce == "colpiv")
    if par is not None:
        line["parity_vs_stored_oracle"] = par
    lam_true = getattr(payload, "lam_true", None)
    if lam_true is not None:   # config 1: the closed-form spectrum lambda = alpha^2 / beta^2
        lt, la = np.sort(np.asarray(lam_true)), np.sort(lam_h.numpy())
        err = float(np.max(np.abs(la - lt) / np.abs(lt))) if la.shape == lt.shape else None
        line["parity_vs_known_spectrum"] = {"max_rel_lambda_err": err, "tol": 1e-9,
                                            "within_tol": err is not None and err <= 1e-9}
    if not args.no_cpu_baseline and ws == 1:
        cb, err = cpu_baseline_fresh_process(args.config, sweeps, args.ref_budget)
        if cb is None:
            F0, J0, G0 = oracle_factors(kind, payload, args.config)
            cb = cpu_baseline_sample(F0, J0, G0, args.config, sweeps, budget_s=args.ref_budget)
            cb["process"] = f"bench process (fresh-process sample failed: {err})"
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--variant", default="bo", choices=["pointwise", "bo", "fb"])
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--nblocks", type=int, default=0)
    ap.add_argument("--ordering", default="hier", choices=["hier", "rr", "level3"],
                    help="block ordering of the blocked variants (DESIGN.md 6, reading R2-5)")
    ap.add_argument("--super-blocks", type=int, default=0, help="super blocks of hier / level3 (0: 2 N, 4 on one GPU)")
    ap.add_argument("--max-sweeps", type=int, default=64,
                    help="C_max; config 3 (S condition 1e12) needs ~36 sweeps, beyond the paper's usual 30")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reduce", default="recipe", choices=["recipe", "colpiv"],
                    help="Phase 2 as the config's recipe says, or the column-pivoted QR path for any "
                         "atoms config (untimed preprocessing, reported as phase2_seconds)")
    ap.add_argument("--want-x", action="store_true",
                    help="also accumulate Z'^{-1} during the sweep (full GHSVD X, NEXT-1)")
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--ref-sweeps", type=int, default=0,
                    help="sweep count used to extrapolate the oracle sample in --impl reference "
                         "(0 = the GPU solve's count for the config, REF_SWEEPS)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    ws = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if args.gpus > 1 and ws == 0:
        # not under torchrun: launch one process per GPU ourselves, or fail loudly
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) visible\n")
            return 2
        return subprocess.call(launch_cmd(args.gpus, sys.argv[1:], _free_port()))
    if ws and ws != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}\n")
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
