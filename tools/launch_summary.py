"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split("(")[0][:48]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for k, v in agg.items() if "ffma_peak" not in k)
print("| kernel | launches | total us | mean us | share (excl. ffma_peak) |\n|---|---|---|---|---|")
for k, (n, t) in agg.items():
    sh = "-" if "ffma_peak" in k else f"{100 * t / tot:.1f}%"
    print(f"| {k} | {n} | {t / 1e3:.1f} | {t / n / 1e3:.2f} | {sh} |")
