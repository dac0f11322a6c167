"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares: python tools/summarize_launches.py launches.csv"""
import csv, re, sys, collections

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").strip()
    name = re.sub(r"<unnamed>::|unnamed>::|hdp::", "", name)
    v = float(r[iv].replace(",", ""))
    unit = hdr[iv + 1] if False else None
    tot[name] += v; cnt[name] += 1
allt = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total':>12s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:12.1f} {100 * v / allt:6.1f}%")
print(f"{'(all)':60s} {sum(cnt.values()):8d} {allt:12.1f}")
