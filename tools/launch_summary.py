"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list per
kernel (dev tool): python tools/launch_summary.py launches.csv [title]"""
import collections
import csv
import re
import sys


def main(path, title=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    to_ms = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").strip()
        name = re.sub(r"<(.*)>", lambda m: "<" + m.group(1).replace("true", "1").replace("false", "0") + ">", name)
        v = float(r[vi].replace(",", "")) * to_ms[r[ui]]
        tot[name][0] += 1
        tot[name][1] += v
    scale = 1.0
    n = sum(v[0] for v in tot.values())
    ms = sum(v[1] for v in tot.values()) * scale
    if title:
        print(title)
    print(f"# launches: {n}   sum of kernel durations: {ms:.1f} ms")
    print(f"{'kernel':52s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>8s}")
    for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:52]:52s} {c:8d} {t * scale:10.2f} {t * scale / ms:7.3f} {t * scale * 1e3 / c:8.1f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
