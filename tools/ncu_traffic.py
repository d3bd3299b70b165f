"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and
duration from `ncu --set full` captures -> profiles/ncu_traffic.json, read by
bench.py for roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/ncu_k_gemv_reg.ncu-rep [...]"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def b(k):
        return float(d[k].replace(",", "")) * scale.get(u[k], 1)

    return {"kernel": d["Kernel Name"].split("(")[0], "grid": d.get("launch__grid_size"),
            "dram_bytes": b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
            "duration_us": float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "nsecond" else 1),
            "source": os.path.basename(path)}


if __name__ == "__main__":
    res = [one(p) for p in sys.argv[1:]]
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))
