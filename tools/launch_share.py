"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares, markdown.
    python tools/launch_share.py gpurun_out/launches.csv > profiles/rNN_launches.md"""
import collections
import csv
import sys


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:90]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
        tot[short] = tot.get(short, 0.0) + v * scale
        cnt[short] += 1
    s = sum(tot.values()) or 1.0
    print(f"# ncu launch list: `{path}`\n")
    print(f"{sum(cnt.values())} launches, {s:.2f} ms total (serialised, cold-cache)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / s:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
