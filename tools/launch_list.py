"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel kind, launches and mean/total time, plus each kind's share of the
sum over our kernels.  Usage: python tools/launch_list.py LAUNCHES.csv [runs]"""
import csv
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_traffic import kind_of  # noqa: E402


def main(path, runs=None):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rd = list(csv.reader(lines))
    h = rd[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    acc, order = {}, []
    for r in rd[1:]:
        k = kind_of(r[ki])
        if k is None:
            continue
        t = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                                              "nsecond": 1e-3}.get(r[ui], 1.0)
        if k not in acc:
            order.append(k)
        s, c = acc.get(k, (0.0, 0))
        acc[k] = (s + t, c + 1)
    tot = sum(s for s, _ in acc.values())
    div = float(runs) if runs else 1.0
    print(f"{'kernel':14s} {'launches':>9s} {'mean_us':>9s} {'us/run':>9s} {'share':>7s}")
    for k in sorted(acc, key=lambda k: -acc[k][0]):
        s, c = acc[k]
        print(f"{k:14s} {c / div:9.1f} {s / c:9.2f} {s / div:9.1f} {100 * s / tot:6.1f}%")
    print(f"{'sum':14s} {'':9s} {'':9s} {tot / div:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
