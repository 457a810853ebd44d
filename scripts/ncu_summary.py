"""Summarise ncu --set full reports: python scripts/ncu_summary.py name=report.ncu-rep ... > json"""
import csv, json, subprocess, sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "s": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__ops_path_tensor_src_fp16_dst_fp32.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        # L2 (LTS) load: throughput against its peak and sectors moved (the L2 -> SM feed of the narrow
        # and batched tiles)
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum", "lts__t_sectors_op_read.sum",
        "lts__t_sectors_op_write.sum", "lts__cycles_elapsed.avg.per_second",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out = {}
for arg in sys.argv[1:]:
    name, path = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            try:
                val = float(v[i].replace(",", ""))
            except ValueError:
                continue
            d[k] = val * UNIT.get(u[i], 1)
    out[name] = d
print(json.dumps(out, indent=1))
