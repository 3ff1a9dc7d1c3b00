"""Average duration per kernel (name prefix up to '<' or '(') from an ncu --metrics
gpu__time_duration.sum --csv launch list: python tools/exp/launch_avg.py LIST.csv [LIST2.csv ...]"""
import csv, sys, collections
for path in sys.argv[1:]:
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in csv.DictReader(lines[start:]):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        v = v / 1e3 if r["Metric Unit"] in ("ns", "nsecond") else (v * 1e3 if r["Metric Unit"] in ("ms", "msecond") else v)
        k = r["Kernel Name"]
        k = k.split("(")[0] if "<" not in k else k[:k.index(">") + 1]
        tot[k] += v
        cnt[k] += 1
    print("##", path)
    for k in sorted(tot, key=lambda k: -tot[k])[:8]:
        print("  %-60s n=%5d avg %9.1f us total %9.1f ms" % (k[-60:], cnt[k], tot[k] / cnt[k], tot[k] / 1e3))
