"""Summarise ncu reports (read here, no GPU): one row per profiled launch with
duration, DRAM traffic, tensor-pipe / XU / FMA / ALU utilisation, occupancy and
registers, plus the top warp-stall reasons. Writes markdown to stdout.

    python tools/ncu_summary.py gpurun_out/ncu_r01_attn.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

M = [("gpu__time_duration.sum", "time"),
     ("dram__bytes_read.sum", "dram rd"),
     ("dram__bytes_write.sum", "dram wr"),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
     ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %"),
     ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %"),
     ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU %"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %"),
     ("launch__registers_per_thread", "regs"),
     ("launch__grid_size", "grid"),
     ("sm__cycles_elapsed.avg.per_second", "SM clk")]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    print("| kernel | " + " | ".join(n for _, n in M) + " | top stalls (share of samples) |")
    print("|---|" + "---|" * len(M) + "---|")
    for path in sys.argv[1:]:
        hdr, units, rows = raw(path)
        ix = {h: i for i, h in enumerate(hdr)}
        stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        for r in rows:
            name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            cells = []
            for m, _ in M:
                cells.append(f"{r[ix[m]]} {units[ix[m]]}".strip() if m in ix else "-")
            tot = sum(float(r[ix[h]] or 0) for h in stall) or 1.0
            top = sorted(((float(r[ix[h]] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall),
                         reverse=True)[:4]
            st = ", ".join(f"{k} {v / tot * 100:.0f}%" for v, k in top if v)
            print(f"| {name} | " + " | ".join(cells) + f" | {st} |")


if __name__ == "__main__":
    main()
