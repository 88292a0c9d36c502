"""Summarise a GHSVD_TRACE launch timeline (blocked sweep, first sweep).

usage: python tools/trace_summary.py trace.csv
Per block step (average over steps): span of each kernel class from the first CTA start
to the last CTA end, and the step period; then the fraction of the sweep during which
no Gram / update kernel (the throughput-bound work) was running."""
import collections
import csv
import sys

rows = list(csv.DictReader(open(sys.argv[1])))
by = collections.defaultdict(dict)
for r in rows:
    by[int(r["step"])][r["kernel"]] = (int(r["start_ns"]), int(r["end_ns"]))
steps = sorted(by)
acc = collections.defaultdict(list)
for s in steps:
    for k, (b, e) in by[s].items():
        acc[k].append((e - b) / 1e3)
print("kernel      mean span [us]")
for k in sorted(acc):
    v = acc[k]
    print(f"{k:10s} {sum(v) / len(v):9.1f}")
ends = [max(e for _, e in by[s].values()) for s in steps]
per = [(ends[i + 1] - ends[i]) / 1e3 for i in range(len(ends) - 1)]
print(f"step period mean {sum(per) / len(per):.1f} us over {len(per)} steps")
# throughput-busy intervals (gram*, update*) vs the sweep span
iv = sorted((b, e) for s in steps for k, (b, e) in by[s].items() if k.startswith(("gram", "update")))
busy, cur_b, cur_e = 0, None, None
for b, e in iv:
    if cur_e is None or b > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_b
        cur_b, cur_e = b, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_b
span = max(ends) - min(b for s in steps for (b, _) in by[s].values())
print(f"sweep span {span / 1e6:.2f} ms, Gram/update running {100.0 * busy / span:.1f} % of it")
