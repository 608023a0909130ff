"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: count, total and mean device time, share of the profiled launches.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/<name>.txt
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
unit = h.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[kn])
    name = re.sub(r"^void ", "", name)[:90]
    v = float(r[mv].replace(",", ""))
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
    v *= scale.get(r[unit], 1.0)
    tot[name] += v                    # nanoseconds
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"launches {sum(cnt.values())}  total device time {all_ns / 1e3:.1f} us "
      f"(serialised by ncu: shares, not absolutes)")
for name, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{name:90s} n={cnt[name]:6d} total_us={v / 1e3:10.1f} avg_us={v / cnt[name] / 1e3:8.2f} "
          f"share={v / all_ns:.3f}")
