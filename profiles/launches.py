"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into the
per-step kernel shares: python profiles/launches.py <launches.csv> <calls>
(<calls> = sc_partition_frames calls the profiled command made)."""
import collections
import csv
import re
import sys


def main():
    path, calls = sys.argv[1], int(sys.argv[2])
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        name = re.sub(r"^cub::\S*?(Device\w+Kernel)\S*", r"cub::\1", name)
        tot[name] += float(r[vi].replace(",", "")) / 1e3
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"# launch list: {path}  ({sum(cnt.values())} launches over {calls} calls, "
          f"{sum(cnt.values()) / calls:.1f} launches per call)")
    print("| kernel | launches/call | us/call (cold, serialised) | share |")
    print("|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| {k} | {cnt[k] / calls:.1f} | {v / calls:.1f} | {100 * v / all_us:.1f}% |")


if __name__ == "__main__":
    main()
