"""Copy the round-end bench lines and ncu outputs from gpurun_out/ into profiles/
(bench lines, ncu --set full summary, launch list, DRAM traffic per step, stall lines)."""
import csv, io, json, os, shutil, statistics, subprocess, sys

R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")
for f in ["r2_bench_8b", "r2_bench_8b_async_estimators", "r2_bench_cfg1_refplan", "r2_bench_llama2_70b_full_t4.0",
          "r2_bench_llama2_7b_t3.5", "r2_bench_llama2_7b_t4.5"]:
    shutil.copy(os.path.join(G, f + ".jsonl"), P)
shutil.copy(os.path.join(G, "launches_r2b.csv"), os.path.join(P, "r2_engine_launches.csv"))
det = subprocess.run(["ncu", "-i", os.path.join(G, "eng_r2b.ncu-rep"), "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
iS, iM, iU, iV = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
want = [("GPU Speed Of Light Throughput", "Memory Throughput"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
        ("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
        ("Compute Workload Analysis", "Executed Ipc Active"), ("Compute Workload Analysis", "Issue Slots Busy"),
        ("Memory Workload Analysis", "Memory Throughput"), ("Memory Workload Analysis", "L1/TEX Hit Rate"),
        ("Memory Workload Analysis", "L2 Hit Rate"), ("Scheduler Statistics", "No Eligible"),
        ("Scheduler Statistics", "Eligible Warps Per Scheduler"), ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
        ("Launch Statistics", "Registers Per Thread"), ("Launch Statistics", "Dynamic Shared Memory Per Block"),
        ("Occupancy", "Achieved Occupancy")]
seen, res = set(), []
for r in rows[1:]:
    if (r[iS], r[iM]) in want:
        o = f"{r[iS]:<32} {r[iM]:<45} {r[iV]} {r[iU]}"
        if o not in seen:
            seen.add(o)
            res.append(o)
open(os.path.join(P, "r2_engine_ncu_full_summary.txt"), "w").write(
    "\n".join(res) + "\n# round-end engine (decode_greedy(4) launch of tools/ncu_engine.py: Llama-3-8B DP 3.5, f16 G), "
    "ncu --set full --clock-control none\n")
txt = open(os.path.join(G, "launches_r2b.csv")).read()
lines = [l for l in txt.splitlines() if l.startswith('"')]
rr = list(csv.reader(io.StringIO("\n".join(lines))))
hh = rr[0]
iid, iM2, iV2 = hh.index("ID"), hh.index("Metric Name"), hh.index("Metric Value")
d = {}
for r in rr[1:]:
    d.setdefault(int(r[iid]), {})[r[iM2]] = float(r[iV2].replace(",", ""))
steps = [v for v in d.values() if 1.4e6 < v["gpu__time_duration.sum"] < 2.5e6]
rd = statistics.median(v["dram__bytes_read.sum"] for v in steps)
wr = statistics.median(v["dram__bytes_write.sum"] for v in steps)
alg = json.loads(open(os.path.join(P, "r2_bench_8b.jsonl")).read())["roofline"]["alg_bytes_per_step"]
json.dump({"bytes_per_step": rd + wr, "read_bytes_per_step": rd, "write_bytes_per_step": wr,
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, median over the "
                     f"{len(steps)} single-step engine_kernel launches of `bench.py --steps 4 --warmup 3 --skip-static` "
                     "(profiles/r2_engine_launches.csv), round 2 end",
           "alg_bytes_per_step": alg, "ratio_to_algorithmic": (rd + wr) / alg},
          open(os.path.join(P, "engine_traffic.json"), "w"), indent=1)
out = subprocess.run([sys.executable, os.path.join(R, "tools", "ncu_lines.py"), os.path.join(G, "eng_r2b.ncu-rep"),
                      os.path.join(R, "paper_2508_06041_b200", "libdpq_b200.so"), "engine_kernel", "25"],
                     capture_output=True, text=True).stdout
open(os.path.join(P, "r2_engine_stall_lines.txt"), "w").write(out)
print(res[2], (rd + wr) / alg, len(steps))
