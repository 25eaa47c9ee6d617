"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

    python tools/ncu_summary.py gpurun_out/launches.csv [top]
prints: kernel, launches, total ms, share of the listed time, mean us per launch.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    n = re.sub(r"\(.*", "", name)              # drop the argument list
    n = re.sub(r"^.*::", "", n) if "::" in n and "<" not in n else n
    n = re.sub(r"rsf::\(anonymous namespace\)::", "", n)
    return n.strip()


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r and "Metric Value" in r:
                hdr = {k: i for i, k in enumerate(r)}
            continue
        if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[hdr["Metric Unit"]] if "Metric Unit" in hdr else "nsecond"
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        k = short(r[hdr["Kernel Name"]])
        tot[k] += v * scale
        cnt[k] += 1
    T = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>9s} {'total ms':>10s} {'share':>7s} {'mean us':>9s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{k[:70]:70s} {cnt[k]:9d} {v:10.2f} {100 * v / T:6.2f}% {1e3 * v / cnt[k]:9.2f}")
    print(f"{'TOTAL':70s} {sum(cnt.values()):9d} {T:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
