"""Summarises an `ncu --set full` capture of the BOCD update kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --tag r01 [--series 32768 --chunk 1000 --R 1024]

Writes profiles/<tag>_ncu_top_kernel.txt (key metrics, stall reasons, per-warp-cell
instruction mix from the SASS source page) and profiles/ncu_traffic.json (DRAM bytes
per launch, read by bench.py for roofline.traffic).  Run it HERE on the report that
gpurun brought back (ncu -i works without a GPU).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"]


def ncu_csv(rep, *args):
    """ncu -i rep ... --csv; or, for a capture exported on the GPU box (tools/gpu/r02_ncu.sh),
    rep = the path stem and the CSV files <stem>.raw.csv / <stem>.src.csv(.gz)."""
    if not rep.endswith(".ncu-rep"):
        import gzip
        page = "raw" if "raw" in args else "src"
        path = f"{rep}.{page}.csv"
        if not os.path.exists(path):
            path += ".gz"
        opener = gzip.open if path.endswith(".gz") else open
        with opener(path, "rt") as f:
            return list(csv.reader(f))
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--series", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=1000)
    ap.add_argument("--R", type=int, default=1024)
    ap.add_argument("--cmd", default="bench.py --steps 2 --warmup 1 (C3 shape), steady-state launch")
    ap.add_argument("--config", default="C3", help="writes profiles/ncu_traffic_<config>.json for bench.py")
    ap.add_argument("--name", default="", help="file stem: profiles/<tag>_ncu_<name>.txt (default top_kernel)")
    a = ap.parse_args()

    raw = ncu_csv(a.rep, "--page", "raw")
    head, units = raw[0], raw[1]
    row = next(r for r in raw[2:] if any("bocd_" in c for c in r))
    d, u = dict(zip(head, row)), dict(zip(head, units))
    kname = d.get("Kernel Name", "")
    warp_cells = a.series * a.chunk * a.R / 32
    cells = a.series * a.chunk * a.R
    lines = [f"# ncu --set full, {os.path.basename(a.rep)}: {a.cmd}", f"kernel: {kname}"]
    for k in KEYS:
        if k in d:
            lines.append(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
    stalls = []
    for k, v in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
        if m and v not in ("", "n/a"):
            try:
                if float(v) >= 0.02:
                    stalls.append((m.group(1), round(float(v), 3)))
            except ValueError:
                pass
    lines.append("stall reasons (warps per issue-active cycle): " + json.dumps(sorted(stalls)))
    t_ms = float(d["gpu__time_duration.sum"])
    cyc = t_ms * 1e-3 * float(d["sm__cycles_elapsed.avg.per_second"]) * (1e9 if u.get(
        "sm__cycles_elapsed.avg.per_second", "").startswith("G") else 1)
    fp64_thread = sum(float(d.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed", 0))
                      for o in ("dfma", "dadd", "dmul")) * cyc
    lines.append(f"warp instructions per warp-cell (32 cells): {float(d['smsp__inst_executed.sum']) / warp_cells:.2f}")
    lines.append(f"FP64 thread instructions (DFMA+DADD+DMUL) per cell: {fp64_thread / cells:.2f}")
    lines.append(f"shared-memory wavefronts per warp-cell: "
                 f"{float(d['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']) / warp_cells:.2f}")

    src = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    sh = src[1]
    isrc, iex = sh.index("Source"), sh.index("Instructions Executed")
    mix = collections.Counter()
    for r in src[2:]:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split()
        if not op:
            continue
        name = op[0]
        name = "MOV" if name.startswith("IMAD.MOV") or name == "MOV" else name.split(".")[0]
        mix[name] += int(r[iex])
    lines.append("mix per warp-cell: " + ", ".join(f"{k} {v / warp_cells:.2f}" for k, v in mix.most_common(20)))
    rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    algo = a.series * a.chunk * 8 + 2 * 3 * a.series * a.R * 8
    lines.append(f"DRAM traffic per launch = {(rd + wr) / 1e9:.3f} GB (algorithmic: x {a.series * a.chunk * 8 / 1e9:.3f} GB"
                 f" + state in/out 2 x {3 * a.series * a.R * 8 / 1e9:.3f} GB = {algo / 1e9:.3f} GB)")
    txt = "\n".join(lines) + "\n"
    path = os.path.join(ROOT, "profiles", f"{a.tag}_ncu_{a.name or 'top_kernel'}.txt")
    open(path, "w").write(txt)
    json.dump({"kernel": kname, "series": a.series, "chunk": a.chunk, "R": a.R, "bytes_per_launch": rd + wr,
               "units": a.series * a.chunk,
               "source": f"{os.path.relpath(path, ROOT)} ({os.path.basename(a.rep)})"},
              open(os.path.join(ROOT, "profiles", f"ncu_traffic_{a.config}.json"), "w"), indent=1)
    print(txt)


if __name__ == "__main__":
    main()
