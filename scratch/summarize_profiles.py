"""gpurun_out/{launches.csv,dram.csv,prof_k_*.ncu-rep} -> profiles/round1_* summaries
(run here after `gpurun ... bash scratch/profile.sh`)."""
import collections
import csv
import json
import subprocess

OUT = "profiles"


def dram():
    rows = [r for r in csv.reader(open("gpurun_out/dram.csv")) if r and r[0] != "==PROF==" and len(r) > 10]
    hdr = rows[0]
    iK, iM, iV, iU, iID = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[(r[iID], r[iK].split("(")[0].replace("trg::", ""))][r[iM]] = float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
    agg = collections.defaultdict(list)
    for (i, k), m in per.items():
        agg[k].append(m)
    out = {}
    for k, ms in agg.items():
        f = lambda key: sum(m.get(key, 0.0) for m in ms) / len(ms)  # noqa: E731
        out[k] = {"launches": len(ms), "dram_read_bytes": f("dram__bytes_read.sum"),
                  "dram_write_bytes": f("dram__bytes_write.sum"), "duration_s": f("gpu__time_duration.sum")}
    return out


def details(k):
    txt = subprocess.run(["ncu", "-i", f"gpurun_out/prof_{k}.ncu-rep", "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    open(f"{OUT}/round1_{k}_details.csv", "w").write(txt)
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    iN, iV, iU = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
            "Achieved Occupancy", "Registers Per Thread", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Compute (SM) Throughput", "Memory Throughput", "Grid Size", "Block Size",
            "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
    out = {}
    for r in rows[1:]:
        if len(r) > iV and r[iN] in want and r[iN] not in out:
            out[r[iN]] = (r[iV], r[iU])
    # FP64 pipe: the arithmetic roofline the path is closest to
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/prof_{k}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hh, vv = rr[0], rr[2]
        for name, key in (("FP64 pipe inst executed (% of peak, active)",
                           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                          ("FP64 pipe cycles active (% of elapsed)",
                           "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")):
            if key in hh:
                out[name] = (f"{float(vv[hh.index(key)]):.2f}", "%")
    return out


def main():
    subprocess.run(["cp", "gpurun_out/launches.csv", f"{OUT}/round1_launches_c2.csv"], check=True)
    d = dram()
    b, c = d["k_build"], d["k_calibrate"]
    tot = b["dram_read_bytes"] + b["dram_write_bytes"] + c["dram_read_bytes"] + c["dram_write_bytes"]
    json.dump({"dram_bytes_per_launch": tot,
               "what": "dram__bytes_read.sum + dram__bytes_write.sum of k_build + k_calibrate (one tree build, C2), "
                       "ncu --clock-control none, averaged over the builds of `bench.py --steps 1 --warmup 3 --batch 0`",
               "per_kernel": d}, open(f"{OUT}/k_build_dram_bytes.json", "w"), indent=1)
    ks = ("k_build", "k_calibrate", "k_register")
    ms = {k: details(k) for k in ks}
    with open(f"{OUT}/round1_summary.md", "w") as f:
        f.write("# Round 1 ncu summary (C2, `bench.py --steps 1 --warmup 3 --batch 0 --c4 0`, B200, --clock-control none)\n\n")
        f.write("Launch list: `round1_launches_c2.csv` (gpu__time_duration.sum per launch). "
                "Full-set details: `round1_<kernel>_details.csv`.\n\n")
        f.write("| metric | " + " | ".join(ks) + " |\n|---|---|---|---|\n")
        for key in ms["k_build"]:
            f.write(f"| {key} | " + " | ".join(f"{ms[k].get(key, ('-', ''))[0]} {ms[k].get(key, ('', ''))[1]}" for k in ks) + " |\n")
        f.write("\nDRAM bytes per launch (dram__bytes_read.sum + write.sum, averaged over launches):\n\n")
        for k, v in d.items():
            f.write(f"* {k}: read {v['dram_read_bytes'] / 1e6:.2f} MB, write {v['dram_write_bytes'] / 1e6:.2f} MB, "
                    f"{v['duration_s'] * 1e3:.3f} ms\n")
    print(open(f"{OUT}/round1_summary.md").read())


if __name__ == "__main__":
    main()
