"""Summarise an ncu report (--page raw --csv) into one line per launch: kernel, duration,
DRAM bytes, DRAM/SM throughput, occupancy, active threads per warp, registers, FP64 pipe use."""
import csv, io, subprocess, sys, re

METRICS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "thr_per_warp",
    "launch__registers_per_thread": "regs",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cyc_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
    "smsp__inst_executed_pipe_fp64.sum": "fp64_warp_inst",
    "smsp__inst_executed.sum": "warp_inst",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
}
STALL = re.compile(r"smsp__average_warp_latency_issue_stalled_(\w+)\.ratio$|smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$")
FULLNAME = True


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    for d in data:
        name = re.sub(r"\(.*", "", d[idx["Kernel Name"]])
        rec = {"kernel": re.sub(r"(?:hm::|<unnamed>::|\(anonymous namespace\)::)", "", name)}
        for m, k in METRICS.items():
            if m in idx:
                v = d[idx[m]].replace(",", "")
                try:
                    v = float(v)
                    if units[idx[m]] in ("msecond", "ms"):
                        v *= 1e3
                    elif units[idx[m]] in ("nsecond", "ns"):
                        v /= 1e3
                    elif units[idx[m]] in ("Kbyte", "KB"):
                        v *= 1e3
                    elif units[idx[m]] in ("Mbyte", "MB"):
                        v *= 1e6
                    elif units[idx[m]] in ("Gbyte", "GB"):
                        v *= 1e9
                except ValueError:
                    pass
                rec[k] = v
        stalls = {}
        for h, i in idx.items():
            m = STALL.match(h)
            if m:
                try:
                    stalls[m.group(1) or m.group(2)] = float(d[i].replace(",", ""))
                except ValueError:
                    pass
        if stalls:
            rec["stalls_top"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        yield rec


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for rec in rows(p):
            print(rec)
