import sys, random
sys.path.insert(0,'/root/repo')
from oracle import ref, tslo
from paper_2105_13336_b200 import workload as W
from paper_2105_13336_b200.planner import Planner
lib = sys.argv[1]
P = Planner(lib_path=lib)
bad = 0; n = 0; resc = 0; cands = 0
fams = ["vgg16","resnet50","inception_v3","inception_v4","densenet","chain"]
for seed in range(int(sys.argv[2]), int(sys.argv[3])):
    rnd = random.Random(seed)
    kind = rnd.random()
    jobs = []
    nj = rnd.choice([1,1,2,3])
    for k in range(nj):
        if kind < 0.5:
            g, l = ref.random_job(seed * 10 + k)
            g["job_id"] = "r%d_%d" % (seed, k)
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
    try:
        o = tslo.build_plan(jobs, cfg)
    except Exception as e:
        o = {"err": str(e)}
    try:
        p = P.build_plan(jobs, cfg)
    except Exception as e:
        p = {"err": str(e)}
    n += 1
    if "err" in o or "err" in p:
        if o.get("err") != p.get("err"):
            bad += 1; print("seed", seed, "ERRDIFF", o.get("err"), "|", p.get("err"))
        continue
    resc += p["stats"].get("rescored", 0); cands += p["stats"]["candidates"]
    if p["plans_json"] != o["plans_json"] or p["reports_json"] != o["reports_json"] or p["merged_peak_history"] != o["merged_peak_history"]:
        bad += 1; print("seed", seed, "MISMATCH bw", bw, cfg)
print("cases", n, "bad", bad, "rescored", resc, "of candidates", cands)
