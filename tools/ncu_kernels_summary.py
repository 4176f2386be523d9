"""Per-kernel summary of an `ncu --set full` report (every captured launch): duration, DRAM bytes, pipe and
issue utilisation, occupancy and the top warp-stall reasons.  python tools/ncu_kernels_summary.py REP [...]"""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__t_sector_hit_rate.pct", "l2hit%")]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if len(rows) < 3:
            print(rep, "no data")
            continue
        h, units = rows[0], rows[1]
        print(f"== {rep}")
        for r in rows[2:]:
            d = dict(zip(h, r))
            u = dict(zip(h, units))
            name = d.get("Kernel Name", "?").split("(")[0]
            print(f"  {name}")
            parts = []
            for k, lab in KEYS:
                if k in d and d[k] not in ("", "n/a"):
                    parts.append(f"{lab}={d[k]}{u.get(k, '') if lab in ('time', 'dram_rd', 'dram_wr') else ''}")
            print("    " + "  ".join(parts))
            stalls = []
            for k, v in d.items():
                if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                    try:
                        stalls.append((int(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                    except ValueError:
                        pass
            tot = sum(s for s, _ in stalls) or 1
            top = sorted(stalls, reverse=True)[:4]
            print("    stalls: " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in top))


if __name__ == "__main__":
    main()
