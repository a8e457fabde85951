"""profiles/ncu_gemm_traffic.json from an `ncu --set full` capture of one
layer's four Dense GEMMs (QKV, O, gate-up, down in launch order).

    python tools/ncu_gemm_traffic.py gpurun_out/prof_gemm.ncu-rep TOKENS SOURCE
"""
import csv
import io
import json
import subprocess
import sys

rep, tokens, source = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]


def val(row, name):
    v = float(row[h.index(name)].replace(",", ""))
    u = units[h.index(name)]
    return v * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)


shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
out, tot_dram, tot_alg = [], 0.0, 0.0
for i, row in enumerate(rows[2:6]):
    name, n, k = shapes[i]
    rd, wr = val(row, "dram__bytes_read.sum"), val(row, "dram__bytes_write.sum")
    alg = 2.0 * n * k + 2.0 * tokens * (n + k)
    tot_dram += rd + wr
    tot_alg += alg
    out.append({"gemm": name, "n": n, "k": k, "tokens": tokens, "dram_read_mb": rd / 1e6,
                "dram_write_mb": wr / 1e6, "algorithmic_mb": alg / 1e6,
                "traffic_over_algorithmic": round((rd + wr) / alg, 3),
                "ncu_us_cold": float(row[h.index("gpu__time_duration.sum")])})
print(json.dumps({"source": source, "dram_bytes_per_launch": tot_dram / 4,
                  "algorithmic_bytes_per_launch": tot_alg / 4,
                  "note": "mean over one layer's four GEMMs; the LM head is not in the capture",
                  "launches": out}, indent=1))
