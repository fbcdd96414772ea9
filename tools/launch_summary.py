"""Summarise an ncu launch list (gpu__time_duration.sum CSV): time per kernel
name, launch count and share of the total (dev tool).
usage: launch_summary.py launches.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")) * 1e-6; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.3f} {100*v/T:6.2f}%")
print(f"{'total':70s} {sum(cnt.values()):8d} {T:10.3f}")
