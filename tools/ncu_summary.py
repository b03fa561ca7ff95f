"""Key metrics + warp-stall breakdown of an ncu report (--set full)."""
import csv, io, subprocess, sys

KEYS = ["Duration", "Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Mem Busy", "Max Bandwidth"]


def main(path, launch=None):
    """Summary of one launch of the report: `launch` = ncu ID, default the
    longest launch."""
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    idi = hdr.index("ID")
    if launch is None:
        durs = {}
        for r in rows[1:]:
            if r[hdr.index("Metric Name")] == "Duration":
                v = float(r[hdr.index("Metric Value")].replace(",", ""))
                durs[r[idi]] = v * (1e3 if r[hdr.index("Metric Unit")] == "ms" else 1.0)
        launch = max(durs, key=durs.get) if durs else "0"
    launch = str(launch)
    print("launch ID:", launch)
    rows = [hdr] + [r for r in rows[1:] if r[idi] == launch]
    ni, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    kn = hdr.index("Kernel Name")
    print("kernel:", rows[1][kn][:90])
    seen = set()
    for r in rows[1:]:
        if r[ni] in KEYS and r[ni] not in seen:
            seen.add(r[ni])
            print(f"  {r[ni]:38s} {r[vi]:>14s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    names, units = rr[0], rr[1]
    vals = next(r for r in rr[2:] if r[names.index("ID")] == launch)
    want = {}
    for i, n in enumerate(names):
        if n.startswith("smsp__average_warp_latency_issue_stalled_") or n.startswith("smsp__average_warps_issue_stalled_"):
            if n.endswith("_per_issue_active.ratio"):
                try:
                    want[n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = float(vals[i])
                except ValueError:
                    pass
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
                 "l1tex__t_bytes_pipe_lsu_mem_global_op_ldgsts.sum", "lts__t_sectors_srcunit_tex.sum",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                 "sm__throughput.avg.pct_of_peak_sustained_elapsed"):
            print(f"  {n:60s} {vals[i]:>16s} {units[i]}")
    print("  stall reasons (warps per issue-active cycle):")
    for k, v in sorted(want.items(), key=lambda kv: -kv[1])[:10]:
        print(f"    {k:40s} {v:8.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
