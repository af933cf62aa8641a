"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel, in launch order."""
import csv, collections, sys
lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]  # skip program output
rows = [r for r in csv.reader(lines) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
agg = collections.OrderedDict(); tot = 0.0
for r in rows[1:]:
    v = float(r[vi].replace(",", "")) / 1e6
    k = r[ki][:80]; agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += v; tot += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {n:5d} {t:9.3f} ms  {100 * t / tot:5.1f}%  {k}")
print(f"  total {tot:.3f} ms")
