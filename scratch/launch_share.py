"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into per-kernel shares."""
import csv, sys, collections, gzip
f = sys.argv[1]
op = gzip.open if f.endswith(".gz") else open
rows = [r for r in csv.reader(op(f, "rt")) if len(r) > 10]
h = rows[0]
kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    if r[mn] != "gpu__time_duration.sum":
        continue
    v = float(r[mv].replace(",", ""))
    unit = h  # ns in csv
    tot[r[kn][:70]] += v; cnt[r[kn][:70]] += 1
T = sum(tot.values())
print(f"total {T/1e6:.2f} ms over {sum(cnt.values())} launches")
print("| share | total ms | launches | kernel |\n|---|---|---|---|")
for k, v in tot.most_common(25):
    print(f"| {100*v/T:.2f}% | {v/1e6:.2f} | {cnt[k]} | `{k}` |")
