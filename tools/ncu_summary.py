"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py ROUND CONFIG:PATHS:REPORT.ncu-rep [...]
    python tools/ncu_summary.py --launches ROUND launches.csv

For each report: a compact text file profiles/<ROUND>_<report>.txt with the
speed-of-light, pipe, occupancy, stall and DRAM numbers, and an entry in
profiles/ncu_summary.json keyed [config][kernel] with the DRAM bytes of the
launch and the number of paths it processed (bench.py scales it to its own
launches for the roofline "traffic" field).
"""

from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    # tcgen05 (collected with --metrics TENSOR_METRICS beside --set full)
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc_scope_1cta.sum",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
]
# the extra --metrics list for kernels that issue tcgen05 (the names ncu --query-metrics gives on B200)
TENSOR_METRICS = ",".join(k for k in KEYS if "tensor" in k or "_tc_" in k)
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio")


def raw_rows(rep: str):
    """Rows of `ncu -i REP --page raw --csv` (or of that CSV saved on the GPU box)."""
    if rep.endswith(".csv"):
        with open(rep) as f:
            out = f.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def num(s: str) -> float:
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return float("nan")


def summarise(round_: str, config: str, paths: int, rep: str, js: dict) -> None:
    base = os.path.splitext(os.path.basename(rep))[0]
    lines = []
    for d, u in raw_rows(rep):
        kname = d["Kernel Name"]
        short = re.sub(r"^void\s+", "", kname).split("(")[0].split("<")[0].split("::")[-1]
        lines.append(f"kernel: {kname}")
        lines.append(f"  grid {d.get('Grid Size')} block {d.get('Block Size')}  config {config}  paths/launch {paths}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")
        stalls = sorted(((STALL.match(k).group(1), num(v)) for k, v in d.items() if STALL.match(k)),
                        key=lambda x: -x[1])
        lines.append("  stalls (warps per issue-active cycle): " +
                     ", ".join(f"{n}={v:.2f}" for n, v in stalls[:10]))
        rd = num(d.get("dram__bytes_read.sum", "nan"))
        wr = num(d.get("dram__bytes_write.sum", "nan"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(u.get("dram__bytes_read.sum", "byte"), 1)
        wr *= scale.get(u.get("dram__bytes_write.sum", "byte"), 1)
        js.setdefault(config, {})[short] = {
            "paths": paths, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "duration_ms": num(d.get("gpu__time_duration.sum", "nan")) *
            (1e-3 if u.get("gpu__time_duration.sum") == "us" else 1e-6 if u.get("gpu__time_duration.sum") == "ns" else 1),
            "fma_pipe_pct": num(d.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "nan")),
            "issue_active_pct": num(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", "nan")),
            "warps_active_pct": num(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "nan")),
            **({"tensor_pipe_pct": num(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"])}
               if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in d else {}),
            **({"tc_pipe_pct": num(d["sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"])}
               if "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active" in d else {}),
            "source": f"profiles/{round_}_{base}.txt (ncu --set full, {paths} paths)",
        }
    with open(os.path.join(PROF, f"{round_}_{base}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


def launches(round_: str, path: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr = None
    agg: dict[str, list[float]] = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg.setdefault(d["Kernel Name"], []).append(num(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    out = [f"# ncu launch list ({os.path.basename(path)}): per-kernel device time, cold-cache and serialised",
           f"# total {tot / 1e6:.3f} ms over {sum(len(v) for v in agg.values())} launches"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{sum(v) / tot:7.3%}  n={len(v):4d}  {sum(v) / 1e6:10.3f} ms  {k[:150]}")
    name = os.path.splitext(os.path.basename(path))[0]
    with open(os.path.join(PROF, f"{round_}_{name}.txt"), "w") as f:
        f.write("\n".join(out) + "\n")


def main(argv):
    os.makedirs(PROF, exist_ok=True)
    if argv[0] == "--tensor-metrics":
        print(TENSOR_METRICS)
        return
    if argv[0] == "--launches":
        for p in argv[2:]:
            launches(argv[1], p)
        return
    round_ = argv[0]
    jpath = os.path.join(PROF, "ncu_summary.json")
    js = json.load(open(jpath)) if os.path.exists(jpath) else {}
    for spec in argv[1:]:
        config, paths, rep = spec.split(":", 2)
        summarise(round_, config, int(paths), rep, js)
    with open(jpath, "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
