"""Dev tool: where the end-to-end C-ABI step spends its time (C2)."""
import sys, os, time, ctypes as C, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref
from paper_2105_13336_b200 import configs as CF, abi
from paper_2105_13336_b200.planner import Planner
P = Planner(0)
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reqs = CF.requests(name) if name.startswith("C5s") else CF.requests(name)[-1:]
groups = [r.jobs for r in reqs]
cfgs = [r.config(ref.initial_peaks(r.jobs)) for r in reqs]
cfg_arr, ncfg, keep = P._configs(cfgs, len(groups))
descs, arr, offs = P._pack_groups(groups)
NG = len(groups)
res = (C.c_void_p * NG)()
L = P.lib
st = abi.TslStats()
rows = []
for i in range(300):
    t0 = time.perf_counter()
    rc = L.tsl_build_plan_groups(P._ctx, arr, offs, NG, cfg_arr, ncfg, res)
    t1 = time.perf_counter()
    for g in range(NG):
        L.tsl_result_final_merged_peak(res[g])
    L.tsl_result_stats(res[0], C.byref(st))
    for g in range(NG):
        L.tsl_result_destroy(res[g])
    t2 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, st.kernel_ms, st.total_ms, st.prep_ms))
rows = rows[50:]
for k, nm in enumerate(["call_ms", "after_ms", "kernel_ms", "total_ms", "prep_ms"]):
    v = [r[k] for r in rows]
    print(f"{nm:10s} mean {statistics.mean(v):.4f} median {statistics.median(v):.4f} min {min(v):.4f}")
print("h2d", st.h2d_bytes, "d2h", st.d2h_bytes)
