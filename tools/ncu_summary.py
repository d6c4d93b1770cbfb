"""Summarise an ncu --set full capture into the JSON bench.py reads
(dram traffic per launch, pipe utilisation) -- run here on the .ncu-rep.

    python tools/ncu_summary.py gpurun_out/sla.ncu-rep sla_tc_kernel profiles/r02_sla_tc_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, kname, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
data = [r for r in rows[2:] if kname in r[hdr.index("Kernel Name")]]
want = {"dram__bytes_read.sum": "dram_bytes_read", "dram__bytes_write.sum": "dram_bytes_write",
        "gpu__time_duration.sum": "gpu_time", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active":
        "tensor_pipe_active_pct", "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active": "tensor_inst_pct",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
        "launch__registers_per_thread": "registers", "sm__cycles_elapsed.avg.per_second": "sm_hz",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct"}
res = {"kernel": data[0][hdr.index("Kernel Name")][:120], "capture": rep, "launches": len(data)}
for m, key in want.items():
    if m in hdr:
        vals = [float(r[hdr.index(m)].replace(",", "")) for r in data]
        res[key] = sum(vals) / len(vals)
        res[key + "_unit"] = units[hdr.index(m)]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for k in ("dram_bytes_read", "dram_bytes_write"):
    if k in res:
        res[k] *= scale.get(res.pop(k + "_unit"), 1)
res["traffic_bytes"] = res.get("dram_bytes_read", 0) + res.get("dram_bytes_write", 0)
if "gpu_time" in res:
    u = res.pop("gpu_time_unit")
    res["gpu_time_ms_under_ncu"] = res.pop("gpu_time") * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
                                                          "msecond": 1, "ms": 1}[u]
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
