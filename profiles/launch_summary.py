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
        ms = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
        name = r[ik].split("(")[0][:60]
        tot[name] += ms
        cnt[name] += 1
    # eval kernels: launched a multiple of n_evals times (plan-time kernels are listed apart)
    ev = {k for k in tot if cnt[k] % n_evals == 0} if n_evals else set(tot)
    ev_ms = sum(tot[k] for k in ev)
    print(f"{'eval kernel':60s} {'launches':>8s} {'ms/eval':>9s} {'ms/launch':>10s} {'share':>7s}")
    for k in sorted(ev, key=lambda k: -tot[k]):
        print(f"{k:60s} {cnt[k]:8d} {tot[k] / (n_evals or 1):9.3f} {tot[k] / cnt[k]:10.3f} {tot[k] / ev_ms * 100:6.1f}%")
    print(f"{'total (eval kernels, serialised under ncu)':60s} {sum(cnt[k] for k in ev):8d} {ev_ms / (n_evals or 1):9.3f}")
    rest = sorted(set(tot) - ev, key=lambda k: -tot[k])
    if rest:
        print("plan-time kernels: " + ", ".join(f"{k} {tot[k]:.2f} ms" for k in rest))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
