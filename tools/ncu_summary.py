"""Summarise ncu captures into profiles/ (run here, on the CPU side).

  python tools/ncu_summary.py --rep gpurun_out/prof_blk.ncu-rep [--rep ...] \
      [--launches gpurun_out/launches_bench.csv] --out profiles/ncu_summary.json

For every kernel in the --set full reports: duration, DRAM bytes read/written per
launch, DRAM throughput %, FP64 / tensor pipe utilisation, achieved occupancy,
registers.  For the launch list: per-kernel launch count, total and mean device time
and share of the total (cold-cache, serialised times: compare SHARES).
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_cycles_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def kname(s):
    """'void ghsvd::<unnamed>::k_blk_update<false>(ghsvd::<unnamed>::BlkArgs, int)' -> 'k_blk_update'."""
    s = s.replace("(anonymous namespace)", "<unnamed>").split("(")[0]
    s = re.sub(r"^void\s+", "", s)
    s = re.sub(r"<[^<>]*>$", "", s.strip())
    return s.split("::")[-1]


def parse_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": kname(r[hdr.index("Kernel Name")])}
        for i, h in enumerate(hdr):
            for key, name in WANT.items():
                if h == key or (h.startswith(key) and name not in d):
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    d[name] = v * SCALE.get(units[i], 1.0)
        res.append(d)
    return res


def parse_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        except ValueError:
            continue
        name = kname(r[ik])
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "total_s": sum(v), "mean_us": sum(v) / len(v) * 1e6, "share": sum(v) / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    try:
        summary = json.load(open(a.out))
    except Exception:
        summary = {"kernels": {}}
    for rep in a.rep:
        per = collections.defaultdict(list)
        for d in parse_rep(rep):
            d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
            per[d["kernel"]].append(d)
        for k, ds in per.items():
            # several launches of one kernel in a capture (e.g. the F/G and Z' updates of one
            # block step): report the mean over the captured mix, keep each launch
            m = {key: sum(x.get(key, 0.0) for x in ds) / len(ds)
                 for key in ds[0] if isinstance(ds[0][key], float)}
            m["kernel"] = k
            m["captured_launches"] = len(ds)
            m["per_launch"] = [{"duration": x.get("duration"), "dram_bytes": x["dram_bytes_per_launch"],
                                "tensor_cycles_pct": x.get("tensor_cycles_pct")} for x in ds]
            m["source"] = rep
            summary["kernels"][k] = m
    if a.launches:
        summary["launch_list"] = parse_launches(a.launches)
        summary["launch_list_source"] = a.launches
    if a.note:
        summary["note"] = a.note
    json.dump(summary, open(a.out, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
