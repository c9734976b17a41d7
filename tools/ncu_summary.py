"""Summarise an ncu --set full capture into profiles/ (markdown + ncu_summary.json entry).

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep <workload-key> <algorithmic-bytes>
"""
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "launch__waves_per_multiprocessor",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    isrc, iss = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    mn = {}
    tot = 0
    for r in rows[2:]:
        s = int(r[iss] or 0)
        tot += s
        op = r[isrc].split()[0] if r[isrc].split() else "?"
        if op.startswith("@"):
            op = r[isrc].split()[1]
        op = op.split(".")[0]
        mn[op] = mn.get(op, 0) + s
    return tot, sorted(mn.items(), key=lambda x: -x[1])[:10]


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    rep, key, alg = sys.argv[1], sys.argv[2], float(sys.argv[3])
    m = raw(rep)
    dur_ms = float(m["gpu__time_duration.sum"][0]) * (1e-6 if m["gpu__time_duration.sum"][1] == "ns"
                                                     else 1e-3 if m["gpu__time_duration.sum"][1] == "us"
                                                     else 1.0)
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    tot, top = stalls(rep)
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                          capture_output=True, text=True).stdout
    md = [f"# ncu --set full: {key}", "", f"report: `{os.path.basename(rep)}` (gpurun_out, not committed)",
          "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in m:
            md.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    md += ["", f"algorithmic bytes per launch: {alg:.4g}", f"DRAM bytes per launch (read+write): "
           f"{rd + wr:.4g} = {(rd + wr) / alg:.3f} x algorithmic",
           f"achieved algorithmic GB/s under ncu (cold L2, serialized): {alg / dur_ms / 1e6:.0f}",
           "", "SASS evidence: UTMALDG (TMA) present: " + str("UTMALDG" in sass) +
           "; SYNCS (mbarrier) present: " + str("SYNCS" in sass), "",
           f"warp-stall samples by opcode (total {tot}):", ""]
    for op, s in top:
        md.append(f"- {op}: {s} ({100 * s / max(tot, 1):.1f}%)")
    os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
    with open(os.path.join(REPO, "profiles", f"{key}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    sp = os.path.join(REPO, "profiles", "ncu_summary.json")
    d = json.load(open(sp)) if os.path.exists(sp) else {}
    d[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
              "duration_ms_ncu": dur_ms, "algorithmic_bytes": alg,
              "registers": m.get("launch__registers_per_thread", ("?",))[0]}
    json.dump(d, open(sp, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
