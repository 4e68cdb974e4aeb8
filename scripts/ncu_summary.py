"""Curated metric table of an ncu --set full report (one column per profiled launch), for
profiles/*.md.   python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [label ...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("gpc__cycles_elapsed.max", "cycles elapsed"),
    ("gpc__cycles_elapsed.max.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
    ("launch__registers_per_thread", "registers / thread"),
    ("sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "INT8 tensor ops (UTCIMMA) % of dense INT8 peak"),
    ("sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.per_cycle_elapsed", "INT8 ops / cycle / SM (peak 16384)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (avg SM)"),
    ("sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed", "tensor pipe active % (busiest SM)"),
    ("sm__pipe_tensor_cycles_active.min.pct_of_peak_sustained_elapsed", "tensor pipe active % (idlest SM)"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("smsp__cycles_active.avg.pct_of_peak_sustained_elapsed", "SMSP active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("smsp__inst_executed.sum", "instructions executed"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA load bytes (L2 -> SM)"),
    ("lts__t_sectors.sum", "L2 sectors (all)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 throughput %"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_scoreboard"),
]


def main():
    rep = sys.argv[1]
    labels = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    names = [d[hdr.index("Kernel Name")][:60] for d in data] if "Kernel Name" in hdr else [str(i) for i in range(len(data))]
    labels = labels or names
    print("| metric | " + " | ".join(labels) + " |")
    print("|---|" + "---|" * len(labels))
    for key, desc in METRICS:
        if key not in hdr:
            continue
        i = hdr.index(key)
        print(f"| {desc} (`{key}`, {units[i]}) | " + " | ".join(d[i] for d in data) + " |")


if __name__ == "__main__":
    main()
