"""Digest of ncu --set full captures (.ncu-rep) into the JSON kept under profiles/: selected metrics per
captured kernel. Usage: python scripts/ncu_summary.py OUT.json LABEL=path.ncu-rep [...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "gpc__cycles_elapsed.max.per_second",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    for d in data:
        yield {h: (f"{v} {u}".strip() if u else v) for h, u, v in zip(hdr, units, d)}


def main():
    out, kernels = sys.argv[1], []
    for arg in sys.argv[2:]:
        label, rep = arg.split("=", 1)
        for i, k in enumerate(rows(rep)):
            e = {"label": label if i == 0 else f"{label} #{i}", "Kernel Name": k.get("Kernel Name", "")}
            e.update({key: k[key] for key in KEYS if key in k})
            kernels.append(e)
    json.dump({"source": "ncu --set full --clock-control none (scripts/gpu_final.sh)", "kernels": kernels},
              open(out, "w"), indent=1)
    for e in kernels:
        print(e["label"], e["Kernel Name"][:60], e.get("gpu__time_duration.sum"), e.get("dram__bytes_read.sum"))


if __name__ == "__main__":
    main()
