import sys, os
sys.path.insert(0, '/root/repo')
from paper_2105_13336_b200.planner import Planner
from paper_2105_13336_b200 import workload as W
from oracle import tslo
P = Planner(0)
jobs = [W.c4_job(70)]
init = sum(tslo.initial_peaks(jobs).values())
cfg = {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": init * 7 // 10}
P.build_plan(jobs, cfg)
p = P.build_plan(jobs, cfg)
s = p["stats"]
print("kernel", s["kernel_ms"], "evalprof", list(s["evalprof"]))
print("inc phases base/new+init/merges/atomics/scans/scatter1/scatter2:", list(s["stageprof"])[:11], "swap pre: maxsize/collect/sort/rest", list(s["stageprof"])[11:15], "phaseA", s["stageprof"][15], "spec", s["cyc_spec"], "conflict", s["cyc_conflict"])
sp = list(s["stageprof"])
print(f"component runs: {sp[18]} runs, {sp[17]} members, sum of per-pass longest run {sp[16]} members, "
      f"sum of per-pass slowest run {sp[19]} cyc, all runs {sp[20]} cyc; A2 total {s['cyc_spec'] - sp[15]} cyc")
print("union-find rounds", sp[23])
