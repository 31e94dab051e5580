"""Summarise an .ncu-rep (read here, no GPU): key throughput, occupancy,
DRAM traffic and warp-stall breakdown.  Usage: python tools/ncu_summary.py rep [rep...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_cycles_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "ffma_thread_inst"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lds_bank_conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main():
    for rep in sys.argv[1:]:
        recs, units = raw(rep)
        for r in recs:
            print(f"== {rep}: {r.get('Kernel Name', '')[:110]}")
            for k, name in KEYS:
                if k in r:
                    print(f"   {name:24s} {r[k]:>16s} {units.get(k, '')}")
            stalls = {k: r[k] for k in r if k.startswith("smsp__average_warp_latency_issue_stalled_")
                      or k.startswith("smsp__pcsamp_warps_issue_stalled_")}
            tot = 0.0
            vals = []
            for k, v in stalls.items():
                if not k.startswith("smsp__pcsamp_warps_issue_stalled_") or k.endswith("_not_issued"):
                    continue
                try:
                    f = float(v.replace(",", ""))
                except ValueError:
                    continue
                tot += f
                vals.append((f, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            if tot:
                print("   stall samples (pc sampling):")
                for f, k in sorted(vals, reverse=True)[:10]:
                    print(f"      {k:28s} {100 * f / tot:5.1f}%")


if __name__ == "__main__":
    main()
