"""Merge `ncu --set full` raw-page CSVs (tools/gpu_round2_final.sh: <dir>/full_<OP>_raw.csv)
into profiles/<tag>_ncu_full_summary.json (one entry per op, replacing re-captured ops) and
copy their details pages to profiles/<tag>_ncu_full_<OP>_details.csv.

  python tools/ncu_full_merge.py gpurun_out/r02f r02
"""
import csv
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "": 1, "usecond": 1, "us": 1, "nsecond": 1e-3,
        "ns": 1e-3, "msecond": 1e3, "ms": 1e3, "Kbyte/block": 1e3, "Mbyte/block": 1e6, "byte/block": 1}
FIELDS = [  # (summary key, metric, scale to the key's unit)
    ("duration_us", "gpu__time_duration.sum", 1),
    ("dram_read_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_write_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("smem_lsu_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    ("smem_tensorcore_wavefronts_pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("smem_dyn_KB", "launch__shared_mem_per_block_dynamic", 1e-3),
]


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    out = {"kernel": data[col["Kernel Name"]]}
    for key, metric, scale in FIELDS:
        if metric not in col:
            continue
        i = col[metric]
        v = float(data[i].replace(",", ""))
        u = units[i]
        if key.endswith("_MB") or key.endswith("_KB"):
            v *= UNIT.get(u, 1)
        elif key == "duration_us":
            v *= UNIT.get(u, 1)
            scale = 1
        out[key] = round(v * scale, 3)
    return out


def main(src, tag):
    dst = os.path.join(ROOT, "profiles", f"{tag}_ncu_full_summary.json")
    summ = json.load(open(dst)) if os.path.exists(dst) else {"how": "", "kernels": {}}
    for raw in sorted(glob.glob(os.path.join(src, "full_*_raw.csv"))):
        op = os.path.basename(raw)[len("full_"):-len("_raw.csv")]
        summ["kernels"][op] = summarise(raw)
        det = os.path.join(src, f"full_{op}_details.csv")
        if os.path.exists(det):
            shutil.copy(det, os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{op}_details.csv"))
        print(op, json.dumps(summ["kernels"][op]))
    with open(dst, "w") as fh:
        json.dump(summ, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
