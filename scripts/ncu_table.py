"""Summarises an ncu --set full capture of one AlexNet INT8 forward (16 launches, see
scripts/gpu_final_r3.sh): writes profiles/ncu/<tag>_forward_table.md and the per-launch DRAM
traffic bench.py reports as roofline.traffic (profiles/ncu/traffic_alexnet_int8.json).
usage: python scripts/ncu_table.py gpurun_out/<tag>_full.ncu-rep <tag> [layer,names,...]"""
import csv
import io
import json
import os
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
if rep.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` exported on the GPU box
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {k: i for i, k in enumerate(hdr)}


def get(r, k):
    try:
        return float(r[col[k]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


# layer of each launch, in plan order (argv[3] overrides; conv1 + relu1 + pool1 run in the
# front kernel, norm1 as an LRN-only pool_lrn pass; fc8 splits K, so a finalize follows it)
names = (sys.argv[3].split(",") if len(sys.argv) > 3 else
         ["data", "conv1", "norm1", "conv2", "pool2", "conv3", "conv4", "conv5", "pool5", "fc6", "fc7", "fc8",
          "fc8_finalize", "fc8_to_fp32"])
lines = ["| layer | kernel | us | dram read MB | dram write MB | UMMA dense % | dram % | SM % |",
         "|---|---|---|---|---|---|---|---|"]
traffic = {}
for name, r in zip(names, data):
    k = r[col["Kernel Name"]][:48]
    us = get(r, "gpu__time_duration.sum")
    if units[col["gpu__time_duration.sum"]] == "ns":
        us /= 1000.0
    elif units[col["gpu__time_duration.sum"]] == "ms":
        us *= 1000.0
    rd = get(r, "dram__bytes_read.sum")
    wr = get(r, "dram__bytes_write.sum")
    # tcgen05 UMMA utilisation: ncu's utcimma / utchmma op counters are normalised to the
    # 2:4-sparse peak; x2 gives the dense fraction (validated: scripts/int8_peak.cu's
    # back-to-back MMA kernel reads 49.9 % -> 99.8 %, profiles/ncu/r2b_umma_counter_validation.csv).
    # (sm__pipe_tensor_cycles_active does not count tcgen05 work.)
    ten = 2 * max(get(r, "sm__ops_path_tensor_op_utcimma_src_int8_realtime.avg.pct_of_peak_sustained_elapsed"),
                  get(r, "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_realtime.avg.pct_of_peak_sustained_elapsed"),
                  0.0)
    dr = get(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    sm = get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
    # units: ncu reports bytes in the unit row (byte / Kbyte / Mbyte)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units[col["dram__bytes_read.sum"]], 1)
    wr *= scale.get(units[col["dram__bytes_write.sum"]], 1)
    lines.append(f"| {name} | {k} | {us:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {ten:.1f} | {dr:.1f} | {sm:.1f} |")
    traffic[name] = {"kernel": k, "dram_bytes": rd + wr, "us": us}
os.makedirs("profiles/ncu", exist_ok=True)
with open(f"profiles/ncu/{tag}_forward_table.md", "w") as f:
    f.write(f"ncu --set full --clock-control none, one AlexNet INT8 b256 forward ({rep})\n\n")
    f.write("\n".join(lines) + "\n")
with open("profiles/ncu/traffic_alexnet_int8.json", "w") as f:
    json.dump({"source": f"ncu --set full, profiles/ncu/{tag}_forward_table.md (bench.py alexnet int8 b256)",
               "per_launch": traffic}, f, indent=1)
print("\n".join(lines))
