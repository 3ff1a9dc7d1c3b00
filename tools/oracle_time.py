"""The sequential CPU oracle's whole DI-SOP / DI-CYC solve to ||F||_1 <= 1e-10 on a bench workload,
one host core (taskset to the first allowed core), adjacency build excluded (the paper's Init):
the time-to-tolerance the bench quotes as `oracle_time_to_tol` (profiles/r2/oracle_<cfg>_full.json).
    python tools/oracle_time.py [config]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import digen
import oracle
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
core = min(os.sched_getaffinity(0))
os.sched_setaffinity(0, {core})
out = {"config": cfg, "n": n, "links": int(len(src)), "tol_l1_fluid": 1e-10, "d": 0.85, "cores": 1}
for v in ("sop", "cyc"):
    t = time.time()
    H, F, st = oracle.di(src, dst, n, d=0.85, tol=1e-10, variant=v)
    out["DI-" + v.upper()] = {"seconds": round(st["solve_seconds"], 2), "cycles": st["cycles"],
                              "equivalent_iterations": round(st["diffusions"] / len(src), 3),
                              "GTEPS": round(st["diffusions"] / st["solve_seconds"] / 1e9, 4),
                              "wall_s_incl_build": round(time.time() - t, 1)}
    print(v, out["DI-" + v.upper()], flush=True)
try:
    out["host_cpu"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
except Exception:
    pass
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"oracle_{cfg}_full.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
