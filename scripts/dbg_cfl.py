"""Debug: device CFL vs host CFL step by step (3-D)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_08571_b200 as R
import workloads as W
import oracle
for n, kw in [((20, 18, 16), {}), ((20, 18, 16), dict(kernel="split")), ((130, 70), {})]:
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx)
    for ms in [1, 2, 3, 6, 12]:
        try:
            with R.Domain(n, dx=dx, **kw) as dom:
                dom.set_state(U0)
                t, k = dom.advance_to(0.06, max_steps=ms)
                Ud = dom.get_state()
            with R.Domain(n, dx=dx, **kw) as dom:
                dom.set_state(U0)
                kh = dom.advance_cfl(0.06, max_steps=ms)
                Uh = dom.get_state()
            print(n, kw, ms, t, k, kh, float(np.max(np.abs(Ud - Uh))), flush=True)
        except Exception as e:
            print(n, kw, ms, "ERR", e, flush=True)
