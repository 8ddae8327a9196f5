"""Time the c3 (or SWEEP_CFG) system matvec under environment variants, one
subprocess each. usage: python tools/kron_sweep.py 'KS_KRON_PAIR=0' 'KS_KRON_PAIR=1'"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2311_18461_b200 as ks
cfg = %r
d, p, n_el = {"c3": (3, 2, 64), "c2": (2, 3, 64), "c5": (3, 4, 128), "c5s": (3, 4, 64)}[cfg]
prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el)
A = ks.assemble_system_operator(prob)
n = prob.N_dof
g = np.random.default_rng(1)
r = ks.DeviceVector.from_host(g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n))
y = ks.DeviceVector(n)
A.time(r, y, 3, flush=False)
ms = A.time(r, y, 10, flush=False)
print("RESULT matvec_ms=%%.4f plan=%%s" %% (ms, A.plan_info()))
'''
cfg = os.environ.get("SWEEP_CFG", "c3")
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(cfg, spec, "|", line[0] if line else ("FAILED " + out.stderr[-400:]), flush=True)
