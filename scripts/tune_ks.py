"""Split-k threshold sweep on one workload: V-cycle time and per-level split per
setting (each setting in a fresh process: thresholds are read once)."""
import json, os, subprocess, sys
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
settings = [(4096, 32768), (4096, 65536), (8192, 32768), (2048, 16384), (16384, 65536), (4096, 4096)]
child = r'''
import sys, json, time, torch
sys.path.insert(0, ".")
import paper_2405_05047_b200 as mg
from problems import configs
import pickle
P = pickle.load(open("/tmp/tune_problem.pkl", "rb"))
S = mg.Multigrid(P.levels, P.bs, omega=P.omega, H=P.fine.H)
b = torch.from_numpy(P.b).cuda(); z = torch.zeros_like(b)
for _ in range(5): S.precondition(z, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30): S.precondition(z, b)
e1.record(); torch.cuda.synchronize()
prof = mg.vcycle_profile(S.ctx, z, b, len(P.levels))
print(json.dumps({"vcycle_ms": e0.elapsed_time(e1) / 30, "level_ms": prof["level_ms"]}))
'''
if not os.path.exists("/tmp/tune_problem.pkl") or "--regen" in sys.argv:
    import pickle
    sys.path.insert(0, ".")
    from problems import configs
    P = configs.build(cfg, keep_geometry=False)
    pickle.dump(P, open("/tmp/tune_problem.pkl", "wb"), protocol=4)
for t4, t2 in settings:
    env = dict(os.environ, MGB200_KS4_SLICES=str(t4), MGB200_KS2_SLICES=str(t2))
    out = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    print(t4, t2, line, flush=True)
