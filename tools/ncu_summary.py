"""Summarise ncu output for profiles/ (markdown on stdout).

    python tools/ncu_summary.py full  <report.ncu-rep> [label]   # --set full capture
    python tools/ncu_summary.py launches <launches.csv>            # gpu__time_duration list
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    ("Kernel Name", "kernel"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "mma.sync (HMMA) pipe %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (realtime)"),
    ("sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_on.avg.pct_of_peak_sustained_elapsed",
     "tcgen05 fp16 sparse ops % of peak"),
    ("sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "tcgen05 fp16 dense ops % of peak"),
    ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_on.avg.pct_of_peak_sustained_elapsed",
     "mma.sp bf16 ops % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem: tensor-core operand reads % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem: LSU wavefronts % of peak"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def full(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    print(f"### {label or path}\n")
    print("| metric | value |\n|---|---|")
    for data in rows[2:]:
        for name, nice in FULL_METRICS:
            if name in head:
                i = head.index(name)
                u = units[i].strip()
                print(f"| {nice} | {data[i]}{(' ' + u) if u else ''} |")
    print()


def launches(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000.0 if unit in ("ns", "nsecond") else v * 1000.0 if unit in ("ms", "msecond") else v
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        if len(short) > 90:
            short = short[:87] + "..."
        agg[short].append(us)
    total = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean µs | total µs | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {100 * sum(v) / total:.1f}% |")
    print()


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        launches(sys.argv[2])
