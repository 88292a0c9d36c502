"""Check bench.py's oracle cost model against a MEASURED full oracle solve on the same host.

bench.py's cpu_baseline (and --impl reference) extrapolate a bounded sample of the oracle
with a two-term cost model and the oracle's own per-sweep transformation counts
(DESIGN.md 10).  On the host that wrote tests/golden/c3_oracle_pointwise.json the full
solve was timed, so the model's estimate can be compared with it directly.

  OMP_NUM_THREADS=8 python tools/validate_cpu_model.py [--budget 30]
"""
import argparse
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--budget", type=float, default=30.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "cpu_model_check.json"))
    args = ap.parse_args()
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    kind, payload = b.make_factors(args.config, "numpy")
    F, J, G = b.oracle_factors(kind, payload, args.config)
    cb = b.cpu_baseline_sample(F, J, G, args.config, 36, budget_s=args.budget)
    ref = json.load(open(os.path.join(ROOT, "tests", "golden", f"c{args.config}_oracle_pointwise.json")))
    out = {"model_estimate_s": cb["value"], "measured_full_solve_s": ref["seconds_sweep"],
           "ratio": cb["value"] / ref["seconds_sweep"], "model": cb, "measured_threads": ref["threads"],
           "measured_cpu": ref["cpu_model"], "this_host_cores": b._cores(), "this_host_cpu": b._cpu_model()}
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
