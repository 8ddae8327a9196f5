"""Small d=3 matvec through the JIT path vs the oracle (debug helper)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2311_18461_b200 as ks
from oracle import oracle as O
from helpers import setup_arrays
O.build_oracle()
for (d, p, ne) in [(3, 2, 8), (3, 2, 20), (2, 2, 40), (3, 3, 12)]:
    a = setup_arrays(ks, d, p, ne, ne)
    A = ks.assemble_system_operator(a["prob"])
    K = O.OracleKron(a["dims"], O.system_terms(a, d, 1.0))
    x = O.random_vec(K.N, 5)
    y = A.apply(x)
    yo = K.apply(x)
    print(d, p, ne, float(np.linalg.norm(y - yo) / np.linalg.norm(yo)), flush=True)
