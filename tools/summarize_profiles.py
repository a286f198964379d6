"""Summarise gpurun_out/ ncu artefacts into profiles/ (committed evidence).

    python tools/summarize_profiles.py r01

Writes profiles/<tag>_launches.csv (per-launch device times of the bench
command), profiles/<tag>_kernels.txt (ncu --set full summary per kernel),
profiles/sweep_traffic.json (DRAM bytes per sweep launch for bench.py's
roofline.traffic) and copies the bench JSON lines.
"""
import csv
import io
import json
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    if rep.endswith(".csv"):  # exported on the GPU box (ncu -i rep --page raw --csv)
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    # launch list
    lpath = os.path.join(OUT, "launches.csv")
    if os.path.exists(lpath):
        lines = open(lpath).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        rows = list(csv.DictReader(lines[start:]))
        per = {}
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
            f.write("id,kernel,duration_ns\n")
            for r in rows:
                if r.get("Metric Name") != "gpu__time_duration.sum":
                    continue
                name = r["Kernel Name"].split("(")[0].replace("void ", "")
                v = float(r["Metric Value"].replace(",", ""))
                unit = r.get("Metric Unit", "ns")
                ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
                f.write(f"{r['ID']},{name},{ns:.0f}\n")
                per.setdefault(name, []).append(ns)
        ours = {k: v for k, v in per.items() if k.startswith(("march::", "echo::"))}
        tot = sum(sum(v) for v in ours.values())
        with open(os.path.join(PROF, f"{tag}_launch_shares.txt"), "w") as f:
            f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares)\n")
            f.write("shares over this library's kernels; torch kernels (the on-device initial condition) listed after\n")
            f.write(f"{'kernel':60s} {'launches':>8s} {'mean_ms':>10s} {'share':>7s}\n")
            for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"{k:60s} {len(v):8d} {statistics.mean(v) / 1e6:10.3f} {sum(v) / tot:7.3f}\n")
            f.write("-- not ours (input generation, outside the timed region):\n")
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                if k not in ours:
                    f.write(f"{k[:60]:60s} {len(v):8d} {statistics.mean(v) / 1e6:10.3f}\n")
    # full capture
    rep = os.path.join(OUT, "prof_round.ncu-rep")
    if not os.path.exists(rep):
        rep = os.path.join(OUT, "prof_round.raw.csv")
    if os.path.exists(rep):
        hdr, units, data = raw(rep)
        ix = {h: i for i, h in enumerate(hdr)}
        keys = KEYS
        sweeps = []
        with open(os.path.join(PROF, f"{tag}_kernels.txt"), "w") as f:
            f.write("ncu --set full --clock-control none, 512^3 config 3 (bench workload), first stage\n")
            for d in data:
                name = d[ix["Kernel Name"]]
                f.write(f"== {name}\n")
                for k in keys:
                    if k in ix:
                        f.write(f"   {k:62s} {d[ix[k]]:>16s} {units[ix[k]]}\n")
                st = []
                for h, i in ix.items():
                    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio"):
                        try:
                            st.append((float(d[i]), h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
                        except ValueError:
                            pass
                f.write("   stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]) + "\n")
                if "k_sweep" in name or "k_march" in name:
                    def val(k):
                        u = units[ix[k]]
                        v = float(d[ix[k]].replace(",", ""))
                        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
                    sweeps.append(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
        if sweeps:
            with open(os.path.join(PROF, "sweep_traffic.json"), "w") as f:
                json.dump({"bytes_per_launch": statistics.mean(sweeps), "per_axis": sweeps,
                           "source": f"profiles/{tag}_kernels.txt (ncu --set full, dram__bytes_read+write)"}, f, indent=1)
    # UCT kernels (divb = 2)
    urep = os.path.join(OUT, "prof_uct.raw.csv")
    if os.path.exists(urep):
        hdr, units, data = raw(urep)
        ix = {h: i for i, h in enumerate(hdr)}
        with open(os.path.join(PROF, f"{tag}_kernels_uct.txt"), "w") as f:
            f.write("ncu --set full --clock-control none, 512^3 config 3 with divb = 2 (UCT), first stage\n")
            for d in data:
                f.write(f"== {d[ix['Kernel Name']]}\n")
                for k in KEYS:
                    if k in ix:
                        f.write(f"   {k:62s} {d[ix[k]]:>16s} {units[ix[k]]}\n")
    for fn in ("bench_default.json", "bench_small.json", "gpu.txt"):
        p = os.path.join(OUT, fn)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(PROF, f"{tag}_{fn}"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
