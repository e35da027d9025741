"""Key metrics of ncu --set full reports, one block per profiled launch (dev tool)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("duration", "gpu__time_duration.sum", 1.0),
    ("dram_read", "dram__bytes_read.sum", 1.0),
    ("dram_write", "dram__bytes_write.sum", 1.0),
    ("dram_throughput_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("fmaheavy_pipe_pct", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("issue_active_pct", "sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("registers", "launch__registers_per_thread", 1.0),
    ("smem_per_block", "launch__shared_mem_per_block", 1.0),
    ("stall_math_throttle", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", 1.0),
    ("stall_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", 1.0),
    ("stall_long_scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1.0),
    ("stall_short_scoreboard", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1.0),
    ("stall_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", 1.0),
]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    print(f"== {rep.split('/')[-1]}")
    for r in rows[2:]:
        print(f"  {r[ki].split('(')[0][-60:]}")
        for name, key, scale in KEYS:
            if key in hdr:
                v = r[hdr.index(key)].replace(",", "")
                try:
                    print(f"    {name:24s} {float(v) * scale:.4g} {units[hdr.index(key)]}")
                except ValueError:
                    pass
