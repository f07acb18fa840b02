"""Per-kernel totals and shares from an ncu launch list
(--metrics gpu__time_duration.sum --csv).   python scripts/launch_summary.py launches.csv"""
import collections
import csv
import re
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void gato::", "").replace("gato::", "").replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else v * 1000 if r[ui] == "ms" else v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    probe = {k: v for k, v in agg.items() if k.startswith("k_fp64_peak")}   # roofline-denominator probe, not the step
    ours = {k: v for k, v in agg.items() if k.startswith("k_") and k not in probe}
    tot = sum(a[1] for a in ours.values())
    print(f"# {path}: {sum(a[0] for a in ours.values())} launches of this repo's kernels, {tot:.1f} us "
          f"(cold-cache, serialised under ncu: compare shares)")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share_%':>8s}")
    for k, (n, t) in ours.items():
        print(f"{k[:60]:60s} {n:8d} {t:10.1f} {t / n:9.1f} {100 * t / tot:8.1f}")
    for k, (n, t) in probe.items():
        print(f"# {k}: {n} launches, {t:.1f} us (fp64 peak probe run by bench.py after the timed region; not part of the step)")
    other = {k: v for k, v in agg.items() if not k.startswith("k_")}
    if other:
        print(f"# other (torch copies/fills around the solve): {sum(a[0] for a in other.values())} launches, "
              f"{sum(a[1] for a in other.values()):.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
