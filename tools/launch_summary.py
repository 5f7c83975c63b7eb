"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel totals and shares."""
import csv
import collections
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v/1e6:10.3f} {v/cnt[k]/1e3:10.2f} {v/T:7.4f}")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {T/1e6:10.3f}")
