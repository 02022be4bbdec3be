"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`): per kernel name, launches, total ms and
share of the listed time, for the kernels of the timed evals (used to write profiles/r2/*_summary.txt).

usage: python profiles/launch_summary.py launches.csv [n_evals]
"""
import csv
import sys
from collections import defaultdict


def main(path, n_evals=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= iv or not r[iv]:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        ms = v / 1e6 if unit == "nsecond" else (v / 1e3 if unit == "usecond" else v)
        name = r[ik].split("(")[0][:60]
        tot[name] += ms
        cnt[name] += 1
    all_ms = sum(tot.values())
    per = f" per eval (/{n_evals})" if n_evals else ""
    print(f"{'kernel':60s} {'launches':>8s} {'ms' + per:>16s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        ms = tot[k] / (n_evals or 1)
        print(f"{k:60s} {cnt[k]:8d} {ms:16.3f} {tot[k] / all_ms * 100:6.1f}%")
    print(f"{'total':60s} {sum(cnt.values()):8d} {all_ms / (n_evals or 1):16.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
