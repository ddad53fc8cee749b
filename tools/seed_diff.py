"""Dev tool: run one fuzz_check seed on a library and diff its plan vs the oracle."""
import sys, random, json, difflib
sys.path.insert(0, '/root/repo')
from oracle import ref, tslo
from paper_2105_13336_b200 import workload as W
from paper_2105_13336_b200.planner import Planner
lib, seed = sys.argv[1], int(sys.argv[2])
src = open('/root/repo/tools/fuzz_check.py').read()
# reuse the generator: exec the per-seed body
rnd = random.Random(seed)
fams = ["vgg16","resnet50","inception_v3","inception_v4","densenet","chain"]
kind = rnd.random()
jobs = []
nj = rnd.choice([1,1,2,3])
for k in range(nj):
    if kind < 0.5:
        g, l = ref.random_job(seed * 10 + k); g["job_id"] = "r%d_%d" % (seed, k)
    else:
        fam = rnd.choice(fams)
        g = W.generate_workload(fam, rnd.choice([1, 8, 32]), 0, rnd.randint(2, 30), "j%d" % k)
        l = W.true_latency_table(g, rnd.randint(0, 99))
    jobs.append((g, l))
ip = ref.initial_peaks(jobs)
bw = rnd.choice([1, 2, 4, 16, 64, 256])
cfg = {"pcie_bandwidth": bw, "transfer_setup": rnd.choice([0, 1, 3]),
       "memory_budget": sum(ip.values()) * rnd.choice([3, 5, 7, 9]) // 10}
if rnd.random() < 0.3:
    cfg["max_swap_ratios"] = {g["job_id"]: rnd.choice([0.1, 0.3, 0.5, 1.0]) for g, _ in jobs}
o = tslo.build_plan(jobs, cfg)
p = Planner(lib_path=lib).build_plan(jobs, cfg)
print("cfg", cfg, "jobs", [(g["job_id"], len(g["ops"])) for g, _ in jobs], "rescored", p["stats"]["rescored"])
a = o["plans_json"].splitlines(); b = p["plans_json"].splitlines()
for line in list(difflib.unified_diff(a, b, "oracle", "device", n=1))[:60]:
    print(line)
print("hist oracle", o["merged_peak_history"]); print("hist device", p["merged_peak_history"])
