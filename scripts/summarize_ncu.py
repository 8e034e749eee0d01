"""Summarise an ncu --set full report of the pass kernels into JSON (per
kernel: duration, DRAM bytes, DRAM / tensor / FP64 pipe utilisation,
registers, dynamic shared memory, top warp-stall reasons).
    python scripts/summarize_ncu.py gpurun_out/<tag>/prof_last.ncu-rep out.json "<capture note>" [pass names...]"""
import csv
import io
import json
import subprocess
import sys

rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3]
names = sys.argv[4:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
keys = {"duration_ms": "gpu__time_duration.sum", "dram_read_GB": "dram__bytes_read.sum",
        "dram_write_GB": "dram__bytes_write.sum",
        "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct",
        "regs": "launch__registers_per_thread", "threads": "launch__block_size",
        "smem_dyn_KB": "launch__shared_mem_per_block_dynamic"}
units = dict(zip(hdr, rows[1]))
scale = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6,
         "ms": 1.0, "us": 1e-3, "ns": 1e-6, "GB": 1.0, "MB": 1e-3, "KB": 1e-6}
res = {"capture": note, "note": "ncu replays are cold-cache and serialised: compare shares, not absolutes",
       "kernels": []}
for i, r in enumerate(data):
    d = {"pass": names[i] if i < len(names) else str(i), "kernel": r[hdr.index("Kernel Name")][:80]}
    for k, m in keys.items():
        if m not in hdr:
            continue
        v = r[hdr.index(m)].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            pass
        u = units.get(m, "")
        if isinstance(v, float) and u in scale and (k.endswith("_GB") or k.endswith("_ms")):
            v *= scale[u]
        d[k] = v
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[j] or 0) for j, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
              and r[j].replace(".", "").isdigit()}
    tot = sum(stalls.values()) or 1.0
    d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:4]}
    if "dram_read_GB" in d and "dram_write_GB" in d and "duration_ms" in d:
        d["traffic_GB"] = d["dram_read_GB"] + d["dram_write_GB"]
        d["GBps_cold"] = d["traffic_GB"] / d["duration_ms"] * 1e3
    res["kernels"].append(d)
json.dump(res, open(out, "w"), indent=1)
for d in res["kernels"]:
    print(d["pass"], {k: d.get(k) for k in ("duration_ms", "traffic_GB", "GBps_cold", "dram_pct_peak",
                                            "tensor_pipe_pct", "fp64_pipe_pct", "regs")})
