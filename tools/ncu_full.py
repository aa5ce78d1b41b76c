"""Summarise an `ncu --set full` capture (raw page CSV: ncu -i X.ncu-rep --page raw --csv) per
kernel launch: duration, DRAM bytes, issue/occupancy, top stall reasons; optionally write the
per-kernel DRAM traffic JSON that bench.py's roofline reads (profiles/r*_<config>_ncu_traffic.json).

usage: python tools/ncu_full.py raw.csv [--header TEXT] [--summary OUT.txt] [--traffic OUT.json]
"""
import argparse
import csv
import json
import re

STALLS = ["barrier", "branch_resolving", "dispatch_stall", "drain", "lg_throttle", "long_scoreboard",
          "math_pipe_throttle", "membar", "mio_throttle", "misc", "no_instruction", "not_selected", "selected",
          "short_scoreboard", "sleeping", "tex_throttle", "wait"]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--header", default="")
    ap.add_argument("--summary")
    ap.add_argument("--traffic")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3, "second": 1e6}
    lines = [a.header] if a.header else []
    traffic = {}
    for r in data:
        name = re.sub(r"^void ", "", r[col["Kernel Name"]]).split("(")[0].replace("cls::", "")
        g = lambda k: num(r[col[k]]) * scale.get(units[col[k]], 1.0) if k in col else 0.0
        us = g("gpu__time_duration.sum")   # microseconds (unit row)
        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        st = {s: g(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio") for s in STALLS}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
        thr = g("smsp__thread_inst_executed_per_inst_executed.ratio")
        lines.append(f"{name:24s} ncu_us={us:8.1f} dram_rd={rd / 1e6:9.1f}MB dram_wr={wr / 1e6:9.1f}MB "
                     f"issue%={g('smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f} "
                     f"occ%={g('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} thr/inst={thr:5.2f} "
                     f"regs={int(g('launch__registers_per_thread'))}  stalls: "
                     + ", ".join(f"{k}:{100 * v / tot:.0f}%" for k, v in top))
        rec = traffic.setdefault(name, {"dram_bytes": 0.0, "dram_read": 0.0, "dram_write": 0.0,
                                        "duration_us_ncu": 0.0, "launches": 0})
        rec["dram_bytes"] += rd + wr
        rec["dram_read"] += rd
        rec["dram_write"] += wr
        rec["duration_us_ncu"] += us
        rec["launches"] += 1
    for rec in traffic.values():   # per launch
        k = rec.pop("launches")
        for f in rec:
            rec[f] /= k
    text = "\n".join(lines)
    print(text)
    if a.summary:
        open(a.summary, "w").write(text + "\n")
    if a.traffic:
        json.dump(traffic, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
