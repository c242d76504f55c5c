"""Summarise the round's ncu captures (tools/profile_round.sh) into profiles/: per-kernel key metrics
(text) and ncu_traffic.json (DRAM bytes per launch, read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}  # durations -> microseconds


def rows_of(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return [], [], []
    return rows[0], rows[1], rows[2:]


def main(tag, src="gpurun_out", dst="profiles"):
    out, traffic = [], {}
    for k in ["gather_rope", "attn_tc_kernel", "attn_tc_combine", "gemm_tc", "residual_kernel", "qkv_epilogue"]:
        path = os.path.join(src, f"{tag}_full_{k}.ncu-rep")
        if not os.path.exists(path):
            continue
        h, u, data = rows_of(path)
        for r in data:
            name = r[h.index("Kernel Name")][:100]
            out.append(f"== {name}")
            vals = {}
            for key in KEYS:
                if key in h:
                    i = h.index(key)
                    out.append(f"   {key:70s} {r[i]:>14s} {u[i]}")
                    try:
                        vals[key] = float(r[i].replace(",", "")) * SCALE.get(u[i], 1)
                    except ValueError:
                        pass
            t = vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)
            traffic.setdefault(k, []).append({"dram_bytes": t, "duration_us": vals.get("gpu__time_duration.sum"),
                                              "grid": vals.get("launch__grid_size")})
    if len(traffic.get("gemm_tc", [])) == 4:  # one layer's QKV, O, gate/up, down: bytes per layer
        traffic["gemm_layer"] = [{"dram_bytes": sum(x["dram_bytes"] for x in traffic["gemm_tc"]),
                                  "duration_us": sum(x["duration_us"] or 0 for x in traffic["gemm_tc"]), "grid": None}]
    with open(os.path.join(dst, f"{tag}_ncu_full_summary.txt"), "w") as f:
        f.write("\n".join(out) + "\n")
    with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
        json.dump({"tag": tag, "kernels": traffic}, f, indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
