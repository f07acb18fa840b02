"""Per-kernel summary of `ncu --set full` captures, keyed by workload and kernel, for bench.py's
`roofline.traffic` and DESIGN.md.
    python scripts/ncu_kernels_json.py c2=gpurun_out/a.ncu-rep c3=gpurun_out/b.ncu-rep > profiles/rNN_ncu_kernels.json"""
import csv, json, re, subprocess, sys

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers", "launch__grid_size": "grid", "launch__block_size": "block",
    "sm__inst_executed_pipe_tensor.sum": "tensor_pipe_inst",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_throughput_pct",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ns": 1e-3, "us": 1.0, "ms": 1e3, "msecond": 1e3,
         "usecond": 1.0, "nsecond": 1e-3}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in rows[2:]:
        name = re.sub(r"[<(].*", "", r[idx["Kernel Name"]]).replace("void ", "").replace("gato::", "")
        rec = {}
        for m, key in WANT.items():
            if m in idx and r[idx[m]] not in ("", "n/a"):
                rec[key] = float(r[idx[m]].replace(",", "")) * SCALE.get(units[idx[m]], 1.0)
        rec["dram_bytes_per_launch"] = rec.pop("dram_read", 0.0) + rec.pop("dram_write", 0.0)
        res.setdefault(name, rec)   # first captured launch of each kernel
    return res


if __name__ == "__main__":
    print(json.dumps({a.split("=")[0]: summarise(a.split("=")[1]) for a in sys.argv[1:]}, indent=1))
