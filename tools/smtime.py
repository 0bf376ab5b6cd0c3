"""ncu CSV (gpu__time_duration.sum + sm__cycles_active.sum per launch, one record) -> per-kernel
and per-stage serialised time and SM-time (GPU-ms equivalent = SM-cycles / SMs / clock).
Stage A1 = the launches before the RSVD's first kernel. Usage: smtime.py in.csv out.json [mhz]."""
import csv, json, sys, io

src, dst = sys.argv[1], sys.argv[2]
mhz = float(sys.argv[3]) if len(sys.argv) > 3 else 1965.0
lines = [ln for ln in open(src) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
launch = {}
for r in rows:
    d = launch.setdefault(int(r["ID"]), {"name": r["Kernel Name"].split("(")[0]})
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        d["ns"] = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1)
    elif r["Metric Name"] == "sm__cycles_active.sum":
        d["cyc"] = v
ids = sorted(launch)
first_rsvd = next((i for i in ids if "bt_" in launch[i]["name"] or "sketch_kernel" in launch[i]["name"]), ids[-1] + 1)
tot_ns = sum(launch[i].get("ns", 0) for i in ids)
tot_cyc = sum(launch[i].get("cyc", 0) for i in ids)
kern, stages = {}, {}
for i in ids:
    d = launch[i]
    st = "A1" if i < first_rsvd else "A2-A11"
    for key, tab in ((d["name"], kern), (st, stages)):
        e = tab.setdefault(key, {"launches": 0, "ns": 0.0, "cyc": 0.0})
        e["launches"] += 1
        e["ns"] += d.get("ns", 0)
        e["cyc"] += d.get("cyc", 0)
def fin(tab):
    return {k: {"launches": e["launches"], "ms_serial": e["ns"] / 1e6, "share_serial": e["ns"] / tot_ns,
                "sm_cycles": e["cyc"], "share_sm_time": e["cyc"] / tot_cyc,
                "gpu_ms_equiv": e["cyc"] / 148 / (mhz * 1e3)}
            for k, e in sorted(tab.items(), key=lambda kv: -kv[1]["cyc"])}
out = {"source": src, "how": "one c3 record under ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum "
       "--clock-control none; GPU-ms equivalent = SM-cycles / 148 / sm_max_mhz",
       "total_ms_serial": tot_ns / 1e6, "total_gpu_ms_equiv": tot_cyc / 148 / (mhz * 1e3),
       "stages": fin(stages), "kernels": fin(kern)}
json.dump(out, open(dst, "w"), indent=1)
for k, e in list(out["kernels"].items())[:14]:
    print(f"{e['gpu_ms_equiv']:7.3f} ms-eq {e['ms_serial']:8.3f} ms  x{e['launches']:4d}  {k}")
print("stages:", {k: round(v["gpu_ms_equiv"], 3) for k, v in out["stages"].items()}, "total", round(out["total_gpu_ms_equiv"], 3))
