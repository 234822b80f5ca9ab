"""Summarise an ncu --set full capture of conv_tc_kernel launches into profiles/ncu_conv_summary.json.

  python scripts/ncu_conv_summary.py gpurun_out/stage.ncu-rep resnet50:0:18:8:3
Per launch: gpu__time_duration, dram__bytes_read+write (the roofline `traffic`), TMA bytes landed
in shared memory (L2 -> SM operand traffic), tensor-pipe activity.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rep, key = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0,
         "nsecond": 1e-3, "msecond": 1e3}


def col(name):
    """Column of a metric; ncu prefixes some section metrics (e.g. 'TPC.TriageCompute.')."""
    for i, h in enumerate(hdr):
        if h == name or h.endswith("." + name):
            return i
    return None


def val(r, name):
    i = col(name)
    if i is None:
        return None
    v = r[i].replace(",", "")
    try:
        return float(v) * scale.get(units[i], 1.0)
    except ValueError:
        return None


launches = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if "conv_tc_kernel" not in name and "conv_halo_kernel" not in name:
        continue
    launches.append({
        "us": val(r, "gpu__time_duration.sum"),
        "dram": (val(r, "dram__bytes_read.sum") or 0) + (val(r, "dram__bytes_write.sum") or 0),
        "tma": val(r, "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"),
        # tensor pipe busy on the busiest SM (the kernel runs on a budget of a few SMs, so the
        # all-SM average is diluted by budget/148)
        "tensor_pct": val(r, "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed"),
    })
n = len(launches)
summary = {"launches": n,
           "dram_bytes_per_launch": round(sum(x["dram"] for x in launches) / n),
           "tma_bytes_per_launch": round(sum(x["tma"] or 0 for x in launches) / n),
           "us_per_launch_ncu": round(sum(x["us"] for x in launches) / n, 2),
           "tensor_pct": round(sum((x["tensor_pct"] or 0) * x["us"] for x in launches) /
                               max(1e-9, sum(x["us"] for x in launches)), 2)
           if any(x["tensor_pct"] is not None for x in launches) else None,
           "note": "ncu replays each launch with cold caches and serialised (--cache-control all): dram bytes "
                   "are an upper bound on HBM traffic; durations are not bench values",
           "per_launch": launches}
out = ROOT / "profiles" / "ncu_conv_summary.json"
doc = json.loads(out.read_text()) if out.exists() else {}
doc[key] = summary
out.write_text(json.dumps(doc, indent=1) + "\n")
print(f"{key}: {n} launches, dram {summary['dram_bytes_per_launch'] / 1e6:.2f} MB/launch, "
      f"TMA->smem {summary['tma_bytes_per_launch'] / 1e6:.2f} MB/launch, {summary['us_per_launch_ncu']} us (ncu)")
