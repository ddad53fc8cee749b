"""Per-stage SM-cycle breakdown of the planning kernel (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref
from paper_2105_13336_b200 import configs as CF
from paper_2105_13336_b200.planner import Planner
P = Planner(lib_path=os.environ["TSL_LIB"]) if os.environ.get("TSL_LIB") else Planner(0)
class _Req:  # C4:<micro_batches> -> one GPT-2-medium job
    def __init__(self, M):
        from paper_2105_13336_b200 import workload as W
        from oracle import tslo
        self.jobs = [W.c4_job(M)]
        self.name = f"C4.M{M}"
        self.n_accesses = sum(len(o["inputs"]) + len(o["outputs"]) for o in self.jobs[0][0]["ops"])
        self._init = sum(tslo.initial_peaks(self.jobs).values())

    def config(self, _):
        return {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": self._init * 7 // 10}


class _Edge:  # edge:<case> -> one tests/golden/edge.json build
    def __init__(self, case):
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
        from helpers import edge_jobs, golden
        c = next(c for c in golden("edge") if c["name"] == case)
        self.jobs, self.name, self.n_accesses, self._cfg = edge_jobs(c), case, c["n_accesses"], c["config"]

    def config(self, _):
        return self._cfg


for name in sys.argv[1:] or ["C1", "C2", "C3", "C5s0"]:
    if name.startswith("edge:"):
        reqs = [_Edge(name[5:])]
    else:
        reqs = [_Req(int(name[3:]))] if name.startswith("C4:") else CF.requests(name)
    for req in [reqs[-1]]:
        cfg = req.config(None if name.startswith(("C4:", "edge:")) else ref.initial_peaks(req.jobs))
        P.build_plan(req.jobs, cfg)
        p = P.build_plan(req.jobs, cfg)
        s = p["stats"]
        tot = s["cyc_total"] or 1
        print(f"{req.name} A={req.n_accesses} kernel={s['kernel_ms']:.3f}ms cyc_total={tot} "
              f"seq={s['cyc_sequence']/tot:.2%} eval={s['cyc_evaluate']/tot:.2%} swap={s['cyc_swap']/tot:.2%} "
              f"rc={s['cyc_recompute']/tot:.2%} evals={s['evaluations']} events={s['timeline_events']} "
              f"cands={s['candidates']} queries={s['busy_intervals']} rescored={s['rescored']} "
              f"spec={s['cyc_spec']/tot:.2%} conflict={s['cyc_conflict']/tot:.2%} sweep={s['cyc_sweep']/tot:.2%} "
              f"merge={s['cyc_merge']/tot:.2%} rescore(job0)={s['cyc_rescore']/tot:.2%} D={s['cyc_apply']/tot:.2%}", flush=True)
        print("   eval phases prep/emit/sort1/group+sort2/automaton/scan+max/peak+report:", list(s["evalprof"]), flush=True)
        d = s["debug"]
        print(f"   rescore detail: queries {d[1]} avg {d[0]/max(1,d[1]):.0f} cyc; commits resolve {d[2]} total {d[3]} "
              f"cyc; pend_sort {s['cyc_pendsort']} (folds {s['fitprof'][3]} cyc) append/schedule {list(s['fitprof'])[:2]}", flush=True)
        fp = list(s["fitprof"])
        print(f"   decide: total {fp[4]} bulk {fp[5]} attn-check {fp[6]} hit-mark {fp[7]} attention {fp[8]}", flush=True)
        qp = list(s.get("queryprof", [0] * 16))
        if qp[10]:
            n = qp[10]
            print(f"   re-score queries (TSL_PROF): {n}; per query prologue {qp[0]/n:.0f} open {qp[1]/n:.0f} "
                  f"sweep {qp[2]/n:.0f} cyc, swept {qp[9]/n:.2f}; search cyc/search busy {qp[3]/max(1,qp[6]):.0f} "
                  f"(x{qp[6]/n:.2f}) pend {qp[4]/max(1,qp[7]):.0f} (x{qp[7]/n:.2f}) storage {qp[5]/max(1,qp[8]):.0f} "
                  f"(x{qp[8]/n:.2f})", flush=True)
        if os.environ.get("TSL_CONF_PROF"):
            print("   conflict phases (prof build): clear/maxend/count/prefix1/prefix2/cursors/fill/consider:",
                  list(s.get("queryprof", [0] * 16))[:8], flush=True)
