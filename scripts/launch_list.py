"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X`):
per kernel name the launches, total and mean duration and share of the profiled time.
The per-launch times are cold-cache and serialised (ncu), so only the SHARES are comparable
with the bench's live timing."""
import csv, sys, collections


def main(path, skip_first=0):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        short = name if len(name) < 90 else name[:87] + "..."
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':92s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:92s} {n:8d} {t/1e3:12.1f} {t/n/1e3:10.1f} {t/tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
