import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_07586_b200 as M
from tests.helpers import det_cases
cases = det_cases()
for name, sd, exc, freqs, cfg in cases:
    t = time.time()
    print("start", name, len(freqs), flush=True)
    r = M.solve(M.Scene(sd), exc, freqs, cfg)
    print("done", name, r.stats.rays_launched, r.stats.contributions, f"{time.time()-t:.2f}s", flush=True)
