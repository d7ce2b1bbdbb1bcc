"""Write the judged profile summaries under profiles/ from ncu captures.

  python tools/make_profiles.py ROUND LAUNCH_CSV REP [REP ...]

profiles/<round>_launches.txt   per-kernel summary of the `ncu --metrics
                                gpu__time_duration.sum` launch list (timed region)
profiles/<round>_<kernel>.txt   key metrics + stall breakdown of one `ncu --set full` capture
profiles/ncu_summary.json       machine-readable: per kernel duration, DRAM bytes per
                                launch, issue/IPC/occupancy (bench.py reads `traffic`)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def summarize(rep):
    raw = ncu_csv(rep, "raw")
    h, units, v = raw[0], raw[1], raw[2]
    get = lambda n: num(v[h.index(n)]) if n in h else None  # noqa: E731
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else os.path.basename(rep)
    dur_ns = get("gpu__time_duration.sum")
    unit = units[h.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in h else "ns"
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    bu = units[h.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in h else "byte"
    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
    bu2 = units[h.index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in h else "byte"
    bscale2 = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu2, 1)
    stalls = {}
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            x = num(v[i])
            if x:
                stalls[n[len("smsp__pcsamp_warps_issue_stalled_"):]] = x
    tot = sum(stalls.values()) or 1.0
    det = ncu_csv(rep, "details")
    dh = det[0]
    mi, vi = dh.index("Metric Name"), dh.index("Metric Value")
    d = {}
    for r in det[1:]:
        d.setdefault(r[mi], r[vi])
    kname = name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1].strip()
    return {
        "kernel": kname,
        "duration_us": round(dur_ns * scale, 2) if dur_ns else None,
        "dram_bytes_per_launch": int(rd * bscale + wr * bscale2) if rd is not None and wr is not None else None,
        "issue_slots_busy_pct": num(d.get("Issue Slots Busy")),
        "ipc_active": num(d.get("Executed Ipc Active")),
        "achieved_occupancy_pct": num(d.get("Achieved Occupancy")),
        "registers": num(d.get("Registers Per Thread")),
        "dram_throughput_pct": num(d.get("DRAM Throughput")),
        # pipe utilisation (% of peak sustained while the SM is active) and the
        # shared-memory wavefront share: the issue-bound kernels' roofline
        "pipes_pct": {k: (round(get(m), 1) if get(m) is not None else None) for k, m in (
            ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            ("fma", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            ("alu", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            ("fp64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            ("lsu", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            ("xu", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            ("shared_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            ("dram", "dram__throughput.avg.pct_of_peak_sustained_elapsed"))},
        "warp_instructions": get("smsp__inst_executed.sum"),
        "stalls_pct": {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:8]},
        "report": os.path.basename(rep),
    }


def main():
    rnd, launch_csv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    import launch_summary
    buf = io.StringIO()
    sys.stdout, old = buf, sys.stdout
    try:
        launch_summary.main(launch_csv)
    finally:
        sys.stdout = old
    with open(os.path.join(out_dir, f"{rnd}_launches.txt"), "w") as f:
        f.write("# ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none\n")
        f.write("#   python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras   (timed region only)\n")
        f.write(buf.getvalue())
    summ = {}
    for rep in reps:
        s = summarize(rep)
        summ[s["kernel"]] = s
        short = s["kernel"].split("::")[-1]
        with open(os.path.join(out_dir, f"{rnd}_{short}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{short} -s 2 -c 1\n")
            f.write("#   python tools/prof_step.py   (c2 workload, 3rd training iteration; tools/prof_full.sh)\n")
            for k, val in s.items():
                f.write(f"{k}: {val}\n")
    path = os.path.join(out_dir, "ncu_summary.json")
    old_summ = json.load(open(path)) if os.path.exists(path) else {}
    old_summ.update(summ)
    json.dump(old_summ, open(path, "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
