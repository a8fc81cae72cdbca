"""Summarise an ncu --set full capture of k_fused: key metrics, dynamic
instruction mix per record and stall reasons.  Usage:
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep RECORDS [--json out.json]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "local_load_bytes", "smsp__sass_inst_executed_op_local_ld.sum",
]


def ncu(path, page, extra=()):
    r = subprocess.run(["ncu", "-i", path, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def main():
    path, recs = sys.argv[1], int(sys.argv[2])
    rows = ncu(path, "raw")
    h, u, v = rows[0], rows[1], rows[2]
    out = {"records_per_launch": recs}
    for i, name in enumerate(h):
        if name in KEYS or ("warps_issue_stalled" in name and name.endswith("per_issue_active.ratio")):
            out[name] = (v[i], u[i])
    src = ncu(path, "source", ["--print-source", "sass"])
    hh = src[1]
    iS, iE = hh.index("Source"), hh.index("Instructions Executed")
    cnt = collections.Counter()
    for r in src[2:]:
        if len(r) <= iE:
            continue
        s = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
        op = s.split()[0].split(".")[0] if s else ""
        try:
            cnt[op] += int(r[iE])
        except ValueError:
            pass
    warps = recs / 32.0
    mix = {k: round(c / warps, 1) for k, c in cnt.most_common()}
    fp64 = sum(mix.get(k, 0) for k in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"))
    out["inst_per_record"] = round(sum(cnt.values()) / warps, 1)
    out["fp64_inst_per_record"] = round(fp64, 1)
    out["mix_per_record"] = mix
    rd = float(out["dram__bytes_read.sum"][0]) * (1e9 if "G" in out["dram__bytes_read.sum"][1] else 1e6 if "M" in out["dram__bytes_read.sum"][1] else 1)
    wr = float(out["dram__bytes_write.sum"][0]) * (1e9 if "G" in out["dram__bytes_write.sum"][1] else 1e6 if "M" in out["dram__bytes_write.sum"][1] else 1)
    out["dram_bytes_per_launch"] = rd + wr
    out["dram_bytes_per_record"] = (rd + wr) / recs
    if len(sys.argv) > 4 and sys.argv[3] == "--json":
        with open(sys.argv[4], "w") as f:
            json.dump(out, f, indent=1)
    for k, val in out.items():
        if k != "mix_per_record":
            print(k, val)
    print("mix:", list(mix.items())[:30])


if __name__ == "__main__":
    main()
