"""Coarse-tail sweep: V-cycle time for tail settings (fresh process each)."""
import json, os, pickle, subprocess, sys
sys.path.insert(0, ".")
child = r'''
import sys, json, torch, pickle
sys.path.insert(0, ".")
import paper_2405_05047_b200 as mg
P = pickle.load(open(sys.argv[1], "rb"))
S = mg.Multigrid(P.levels, P.bs, omega=P.omega, H=P.fine.H)
b = torch.from_numpy(P.b).cuda(); z = torch.zeros_like(b)
for _ in range(5): S.precondition(z, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): S.precondition(z, b)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"vcycle_ms": e0.elapsed_time(e1) / 50}))
'''
settings = [("0", "1024", "0"), ("c", "64", "0"), ("c", "128", "0"), ("c", "256", "0"), ("c", "600", "0")]
for cfg in sys.argv[1:]:
    path = f"/tmp/tail_{cfg}.pkl"
    if not os.path.exists(path):
        from problems import configs
        pickle.dump(configs.build(cfg, keep_geometry=False), open(path, "wb"), protocol=4)
    for ks8 in ("256",):
      for tail, sl, ctas in settings:
        env = dict(os.environ, MGB200_TAIL=tail, MGB200_TAIL_SLICES=sl, MGB200_KS8_SLICES=ks8)
        if ctas != "0":
            env["MGB200_TAIL_CTAS"] = ctas
        out = subprocess.run([sys.executable, "-c", child, path], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(cfg, "ks8<", ks8, "tail", tail, "slices<=", sl, line, flush=True)
