"""Loop structure of one kernel's SASS from an ncu source page (--page source --csv --print-source sass):
runs of consecutive instructions with the same execution count (a loop body executes as one run), their
share of the warp-level instructions and stall samples, and their mnemonics; plus thread instructions
per evaluation, counting one MUFU.EX2 per (pixel, entry) evaluation (k_fwd).
usage: python tools/sass_classes.py kfwd_sass.csv [top]"""
import collections
import csv
import sys


def main(path, top=8):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    ie, isrc = h.index("Instructions Executed"), h.index("Source")
    ist = h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((int(r[ie].replace(",", "") or 0), int(r[ist].replace(",", "") or 0), r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    tot_i = sum(d[0] for d in data)
    tot_s = sum(d[1] for d in data) or 1
    runs = []
    for k, d in enumerate(data):
        if runs and runs[-1]["exec"] == d[0] and runs[-1]["end"] == k - 1:
            runs[-1]["end"] = k
            runs[-1]["ops"].append(d[2])
            runs[-1]["stall"] += d[1]
        else:
            runs.append({"exec": d[0], "beg": k, "end": k, "ops": [d[2]], "stall": d[1]})
    for r in sorted(runs, key=lambda r: -r["exec"] * len(r["ops"]))[:top]:
        n = len(r["ops"])
        ops = collections.Counter(o.split()[1] if o.startswith("@") else o.split()[0] for o in r["ops"] if o)
        print(f"run {r['beg']:5d}-{r['end']:5d} n={n:4d} exec/inst={r['exec']:.3e} "
              f"instr share={100 * r['exec'] * n / tot_i:5.1f}% stall share={100 * r['stall'] / tot_s:5.1f}%  "
              f"{dict(ops.most_common(8))}")
    ex2 = sum(d[0] for d in data if "MUFU.EX2" in d[2])
    if ex2:
        print(f"warp instr {tot_i:.4e}  MUFU.EX2 warp instr {ex2:.4e} -> thread evals {ex2 * 32:.4e}; "
              f"instr per eval (thread) {tot_i / ex2:.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
