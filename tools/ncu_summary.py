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
}
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
        yield rec


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for rec in rows(p):
            print(rec)
