"""Summarise the warp-stall samples of an `ncu --page source --csv --print-source sass` export:
samples per stall reason over the whole kernel and the instructions with the most samples."""
import csv
import gzip
import sys


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, ntop=25):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as fh:
        rows = list(csv.reader(fh))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
    seen, uniq = set(), []
    for r in data:  # the export repeats each instruction once per source view
        if r[0] not in seen:
            seen.add(r[0])
            uniq.append(r)
    ws, si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    st = [c for c in h if c.startswith("stall_") and "Not" not in c]
    tot = sum(fl(r[ws]) for r in uniq)
    print(f"instructions {len(uniq)}  executed {sum(fl(r[ie]) for r in uniq):.4g}  stall samples {tot:.0f}")
    for c in sorted(st, key=lambda c: -sum(fl(r[h.index(c)]) for r in uniq)):
        v = sum(fl(r[h.index(c)]) for r in uniq)
        if v > 0.005 * tot:
            print(f"  {c:28s} {v:10.0f}  {100 * v / tot:5.1f}%")
    print("top instructions (samples, executed, source, top reasons)")
    for r in sorted(uniq, key=lambda r: -fl(r[ws]))[:ntop]:
        reasons = sorted(((fl(r[h.index(c)]), c) for c in st), reverse=True)[:2]
        print(f"  {int(fl(r[ws])):7d} {int(fl(r[ie])):10d}  {r[si][:64]:64s} " +
              ", ".join(f"{c[6:]} {int(v)}" for v, c in reasons if v > 0))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
