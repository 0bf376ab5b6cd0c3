"""Summarise an ncu --set full report into profiles/ncu_summary_<tag>.json (kernel -> metrics).
  python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/ncu_summary_r01.json [--merge]"""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
res = json.load(open(out)) if "--merge" in sys.argv else {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
    if name in res and "--merge" not in sys.argv:
        name = name + "#2"
    d = {}
    for k in KEYS:
        if k in hdr:
            v = r[hdr.index(k)].replace(",", "")
            try:
                d[k] = {"value": float(v), "unit": units[hdr.index(k)]}
            except ValueError:
                pass
    res[name] = d
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
