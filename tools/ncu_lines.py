"""Hot CUDA source lines of one kernel from an ncu report:
    ncu -i rep --page source --csv --print-source cuda,sass -k regex:NAME > f.csv
    python tools/ncu_lines.py f.csv [top]
Prints per line: share of warp-level instructions, share of stall samples, average active threads."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ci, ti, si = (hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"),
                  hdr.index("Warp Stall Sampling (All Samples)"))
    lines = []
    for r in rows:
        if len(r) > ci and r[0].isdigit():
            f = lambda i: float(r[i]) if r[i] not in ("", "-") else 0.0
            try:
                lines.append((int(r[0]), r[1].strip()[:110], f(ci), f(ti), f(si)))
            except ValueError:   # a source line whose quotes broke the CSV quoting
                continue
    tot = [sum(x[k] for x in lines) for k in (2, 3, 4)]
    print(f"total warp-instr {tot[0]:.3e} thread-instr {tot[1]:.3e} stall samples {tot[2]:.0f}")
    for ln, s, c, t, st in sorted(lines, key=lambda x: -x[4])[:top]:
        print(f"{ln:>5} {100 * c / max(tot[0], 1):5.1f}%i {100 * st / max(tot[2], 1):5.1f}%s {t / max(c, 1):5.1f}thr  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
