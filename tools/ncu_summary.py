"""Summarize ncu outputs into profiles/<round>/.

    python tools/ncu_summary.py launches <launches.csv> <out.json>
    python tools/ncu_summary.py full <report.ncu-rep> <out.json> [--pixels N --config NAME]

`launches`: per-kernel launch counts, total/avg device time and share of the
profiled time (cold-cache, serialized -- compare shares, not absolutes).
`full`: per kernel the key metrics of an `ncu --set full` capture: duration,
DRAM bytes read/written, DRAM/SM throughput, occupancy, top stall reasons; with
--pixels, DRAM bytes per pixel (bench.py reads profiles/ncu_traffic.json).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path


def short(name: str) -> str:
    name = name.replace("ut::<unnamed>::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0][:90]


def launches(path: str, out: str) -> None:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = short(r[ix["Kernel Name"]])
        agg[k][0] += 1
        agg[k][1] += float(r[ix["Metric Value"]].replace(",", ""))
    total = sum(v[1] for k, v in agg.items() if "synth_kernel" not in k)
    doc = {"note": "ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, "
                   "serialized launches; share excludes the data generator (setup)",
           "kernels": []}
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        doc["kernels"].append({"kernel": k, "launches": n, "total_us": round(t / 1e3, 1),
                               "avg_us": round(t / n / 1e3, 2),
                               "share_of_path": None if "synth_kernel" in k
                               else round(t / total, 4)})
    Path(out).write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
}

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
         "ms": 1e-3, "s": 1.0, "second": 1.0}


def full(rep: str, out: str, pixels: int | None, config: str | None) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    doc = {"report": Path(rep).name, "kernels": []}
    for v in rows[2:]:
        ent = {"kernel": short(v[hdr.index("Kernel Name")])}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    val = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if key in ("dram_read", "dram_write"):
                    val *= SCALE.get(u, 1.0)
                elif key == "duration":
                    val *= SCALE.get(u, 1e-9) * 1e6  # -> us
                ent[key] = val
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and \
                    h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), h[len("smsp__average_warps_issue_stalled_"):
                                                  -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        ent["top_stalls"] = [{"reason": n, "cycles_per_issue": round(x, 2)}
                             for x, n in sorted(stalls, reverse=True)[:5]]
        if "dram_read" in ent and "dram_write" in ent:
            ent["dram_bytes"] = ent["dram_read"] + ent["dram_write"]
            if pixels:
                ent["dram_bytes_per_pixel"] = round(ent["dram_bytes"] / pixels, 2)
        doc["kernels"].append(ent)
    Path(out).write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))
    if pixels and config:
        proj = [k for k in doc["kernels"] if "project" in k["kernel"]]
        if proj:
            tfile = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
            cur = json.loads(tfile.read_text()) if tfile.exists() else {}
            cur[config] = {"kernel": proj[0]["kernel"],
                           "bytes_per_pixel": proj[0].get("dram_bytes_per_pixel"),
                           "source": f"{Path(rep).name}: ncu --set full, {pixels} px launch"}
            tfile.write_text(json.dumps(cur, indent=1) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        args = sys.argv[4:]
        px = int(args[args.index("--pixels") + 1]) if "--pixels" in args else None
        cfg = args[args.index("--config") + 1] if "--config" in args else None
        full(sys.argv[2], sys.argv[3], px, cfg)
