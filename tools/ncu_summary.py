"""Summarise an ncu report: key metrics + top SASS lines by executed instructions."""
import csv, io, subprocess, sys

def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    want = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Achieved Occupancy",
            "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
            "No Eligible", "Static Shared Memory Per Block"]
    seen = set()
    for r in rows[1:]:
        if r[mi] in want and r[mi] not in seen:
            seen.add(r[mi]); print(f"  {r[mi]} = {r[vi]} {r[ui]}")

def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for n in names:
        if n in h:
            print(f"  {n} = {rows[2][h.index(n)]} {rows[1][h.index(n)]}")

def source(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si, ei, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ei and r[ei].isdigit()]
    tot = sum(int(r[ei]) for r in data)
    stall = sum(int(r[wi]) for r in data if r[wi].isdigit())
    print(f"  total warp-instructions {tot/1e6:.2f}M, stall samples {stall}")
    hot = sorted(data, key=lambda r: -int(r[wi]) if r[wi].isdigit() else 0)[:top]
    for r in hot:
        print(f"   {int(r[ei])/1e6:7.2f}M  stall {r[wi]:>6}  {r[si].strip()[:80]}")

rep = sys.argv[1]
print(rep)
details(rep)
raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum"])
if len(sys.argv) > 2:
    source(rep, int(sys.argv[2]))
