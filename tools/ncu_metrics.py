"""Print selected raw metrics of an ncu report (one line per profiled kernel)."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active"]
STALLS = ["long_scoreboard", "barrier", "wait", "sleeping", "mio_throttle", "short_scoreboard", "lg_throttle",
          "selected", "math_pipe_throttle", "branch_resolving", "no_instruction", "dispatch_stall", "membar"]


def main(path, extra=()):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:60]
        out = {}
        for w in list(WANT) + list(extra):
            if w in h:
                out[w.split("__")[-1][:45] if w.count("__") else w] = r[h.index(w)]
        st = {}
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in h:
                st[s] = r[h.index(k)]
        print(name)
        for k, v in out.items():
            print("   ", k, v)
        print("    stalls", st)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
