"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch):
per-kernel totals and shares. Usage: python ncu_summary.py launches.csv"""
import collections
import csv
import io
import re
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def load(path):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(text[start:]))))


def short(name):
    name = re.sub(r"^void ", "", name)
    m = re.match(r"([\w:]+?)(<.*)?\(", name)
    base = m.group(1) if m else name[:60]
    base = re.sub(r"vp::\(anonymous namespace\)::|vp::<unnamed>::|at::native::|at::", "", base)
    tmpl = ""
    if m and m.group(2):
        tmpl = m.group(2)[:60]
    return base + tmpl


def main(path, only_vp=False):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        nm = r["Kernel Name"]
        if only_vp and "vp::" not in nm:
            continue
        v = float(r["Metric Value"]) * SCALE.get(r["Metric Unit"], 1.0)
        k = short(nm)
        agg[k][0] += 1
        agg[k][1] += v
        tot += v
    print(f"{'us':>10} {'share':>6} {'n':>5}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {n:5d}  {k}")
    print(f"total {tot:.1f} us over {sum(n for n, _ in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1], only_vp="--vp" in sys.argv)
