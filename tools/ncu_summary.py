"""Summarise an ncu --set full capture of a fold kernel into the JSON that
bench.py's roofline reads (profiles/<cfg>_fold_ncu_summary.json)."""
import csv, json, subprocess, sys

rep, out, kernel, alg_bytes = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))
u = dict(zip(h, units))


def num(k, scale_to_bytes=False):
    x = float(m[k].replace(",", ""))
    if scale_to_bytes:
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)
    return x


rd, wr = num("dram__bytes_read.sum", True), num("dram__bytes_write.sum", True)
d = {"kernel": kernel, "source": f"{rep} (ncu --set full --clock-control none --import-source on, one launch)",
     "duration_us_under_ncu": num("gpu__time_duration.sum") / (1e3 if u["gpu__time_duration.sum"] == "nsecond" else 1),
     "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
     "algorithmic_bytes_per_launch": alg_bytes, "traffic_over_algorithmic": (rd + wr) / alg_bytes,
     "tensor_pipe_pct_of_peak_elapsed": num("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
     "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
     "lts_throughput_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
     "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
     "smem_tc_wavefronts": num("l1tex__data_pipe_tc_wavefronts_mem_shared.sum"),
     "smem_lsu_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
     "sm_cycles_elapsed_avg": num("sm__cycles_elapsed.avg"),
     "registers_per_thread": num("launch__registers_per_thread"), "grid": num("launch__grid_size")}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
