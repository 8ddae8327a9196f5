"""Time the c3 FD apply under environment variants (one subprocess each, since
layout switches are read at handle creation).
usage: python tools/fd_sweep.py 'KS_FD_AXIS1=0' 'KS_FD_AXIS1=1' ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2311_18461_b200 as ks
cfg = %r
d, p, n_el = {"c3": (3, 2, 64), "c2": (2, 3, 64), "c5s": (3, 4, 64), "c4p2": (2, 2, 128), "c4p3": (2, 3, 128), "c4p4": (2, 4, 128), "c4p5": (2, 5, 128), "c4p6": (2, 6, 128), "c5": (3, 4, 128)}[cfg]
prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el)
P = ks.FDPreconditioner(prob)
n = prob.N_dof
g = np.random.default_rng(1)
r = ks.DeviceVector.from_host(g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n))
z = ks.DeviceVector(n)
P.time(r, z, 3)
ms, mk = P.time(r, z, 20)
print("RESULT total_ms=%%.4f transforms_ms=%%.4f rest_ms=%%.4f info=%%s" %% (ms, mk, ms - mk, P.info()))
'''

cfg = os.environ.get("SWEEP_CFG", "c3")
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(spec, "|", line[0] if line else ("FAILED " + out.stderr[-400:]), flush=True)
