"""Summarise one `ncu --set full` capture of the dominant loss kernel into
profiles/ncu_traffic.json (the `traffic` figure bench.py reports per launch).

    python scripts/ncu_traffic.py gpurun_out/prof_bench_full.ncu-rep --rows 131072 --V 152064 \
        --plan-kernel 3 --capture "<the ncu command line>"
"""
import argparse
import csv
import io
import json
import os
import subprocess

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "%": 1.0}

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--rows", type=int, required=True)
ap.add_argument("--V", type=int, required=True)
ap.add_argument("--plan-kernel", type=int, required=True)
ap.add_argument("--capture", default="")
ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "profiles", "ncu_traffic.json"))
args = ap.parse_args()
raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]


def get(name):
    i = hdr.index(name)
    return float(vals[i].replace(",", "")) * UNIT.get(units[i], 1.0)


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
alg = 4 * args.V + 29  # 2V read, 2V write, 16 B row info, fp64 term + logp + flag
out = {
    "kernel": vals[hdr.index("Kernel Name")],
    "plan_kernel": args.plan_kernel,
    "capture": args.capture,
    "V": args.V,
    "rows": args.rows,
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "dram_bytes_per_row": (rd + wr) / args.rows,
    "algorithmic_bytes_per_row": alg,
    "traffic_over_algorithmic": (rd + wr) / args.rows / alg,
    "duration_ms_under_ncu": get("gpu__time_duration.sum"),
    "dram_throughput_pct_of_peak": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "l2_hit_rate_pct": get("lts__t_sector_hit_rate.pct"),
    "issue_active_pct": get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": get("launch__registers_per_thread"),
}
with open(args.out, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
