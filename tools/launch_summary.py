"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0].replace("tcec::<unnamed>::", "").replace("void ", "")
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[14]) / 1e6
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:70]:70s} launches={n:5d} total_ms={t:10.3f} share={t / tot * 100:6.2f}%")
print(f"TOTAL {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
