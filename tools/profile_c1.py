"""c1 (PEC sphere, one incidence, 4.0 M paths): two launches for ncu (-s 1 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_07586_b200 as M  # noqa: E402

sd = M.make_builtin_scene("sphere", {"subdivisions": 5})
s = M.Scene(sd)
exc = M.monostatic_excitation(90.0, 0.0)
cfg = M.McConfig(strata_per_wavelength=30, samples_per_stratum=1, max_bounce=8, seed=1)
for _ in range(2):
    vals, st = M.estimate_batch(s, [(exc, 0.0)], [[exc]], [10e9], cfg)
print(st.rays_launched, st.kernel_ms)
