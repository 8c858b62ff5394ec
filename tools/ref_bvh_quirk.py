"""The reference's own BVH vs its brute force on the c5 airframe (CPU only):
runs the compiled reference and the oracle restatement on one c5 azimuth at
reduced strata, lists the paths whose contributions differ, rebuilds their
launch rays and traces them with the reference's BVH (mode 0), the
reference's brute force (mode 1) and the oracle.  Finding:
on near-coincident skin surfaces the reference's BVH returns a hit ~1e-14
farther than its brute force; the oracle and the GPU follow brute force.

    python tools/ref_bvh_quirk.py
"""
import sys, numpy as np, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_07586_b200 as M, oracle
from paper_2511_07586_b200.geometry import airframe
from tests.helpers import sort_contribs
sd,_=airframe(1_000_000, seed=5, dielectric_skin=True); sd.eps_imag=None
exc=M.monostatic_excitation(90.0, -5.0)
cfg=M.McConfig(strata_per_wavelength=3, samples_per_stratum=1, max_bounce=24, seed=5, roulette=M.RouletteConfig(enabled=True,q=0.5,min_bounce=3))
freqs=np.linspace(8e9,12e9,128)
t=time.time(); r=oracle.ref_estimate(oracle.ref_scene(sd), exc.to_c(), freqs, cfg.to_c(), 16, True, 1<<22); print('ref', time.time()-t, r['stats'].rays_launched, r['stats'].contributions)
t=time.time(); p=oracle.port_estimate(oracle.port_scene(sd), exc.to_c(), freqs, cfg.to_c(), True, 1<<22); print('port', time.time()-t, p['stats'].contributions)
a=sort_contribs(r['contributions']); b=sort_contribs(p['contributions'])
print(len(a), len(b))
if len(a)==len(b):
    diff = np.nonzero(a['order_key']!=b['order_key'])[0]
    print('key diffs', len(diff))
rel=np.max(np.abs(r['values']-p['values']))/np.max(np.abs(r['values'])); print('values rel', rel)
ka=set(a['order_key'].tolist()); kb=set(b['order_key'].tolist())
only_ref=sorted(ka-kb); only_port=sorted(kb-ka)
print('only ref', len(only_ref), 'only port', len(only_port))
print('bounces only_ref', [k & 0xff for k in only_ref][:20])
print('bounces only_port', [k & 0xff for k in only_port][:20])
cells=sorted(set([k>>8 for k in only_ref+only_port]))
print('paths', len(cells), cells[:10])
# same key, different record?
common = sorted(ka & kb)
ia = {k:i for i,k in enumerate(a['order_key'].tolist())}; ib = {k:i for i,k in enumerate(b['order_key'].tolist())}
nd = sum(1 for k in common if a[ia[k]].tobytes()!=b[ib[k]].tobytes())
print('common keys with different records', nd)
# first-bounce check of the differing paths: launch ray through ref BVH vs brute force
import ctypes as C
L=oracle.port()
L.orc_launch_rect.argtypes=[C.c_void_p, C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double)]
ps_=oracle.port_scene(sd)
out=np.zeros(11); L.orc_launch_rect(ps_.h, oracle.dp(np.array(exc.k_inc, dtype=np.float64)), 0.0, oracle.dp(out))
print('rect', out)
# reconstruct the launch rays of the differing paths (solver_mc.cpp sample_stratum)
import math
c_, u_, v_ = out[0:3], out[3:6], out[6:9]; hu, hv = out[9], out[10]
lam = 299792458.0/12e9; target = lam/3.0
nu = max(1, math.ceil(2*hu/target)); nv = max(1, math.ceil(2*hv/target))
print('nu nv', nu, nv, nu*nv)
os_, ds_ = [], []
for cell in cells:
    i, j = cell % nu, cell // nu
    ju = L.orc_counter_uniform
    ju.restype = C.c_double; ju.argtypes = [C.c_uint64]*5
    uu = ju(5, cell, 0, 0, 0x101); vv = ju(5, cell, 0, 0, 0x102)
    su = -1.0 + 2.0*(i+uu)/nu; sv = -1.0 + 2.0*(j+vv)/nv
    p = (c_ + u_*(su*hu)) + v_*(sv*hv)
    os_.append(p); ds_.append(np.array(exc.k_inc))
os_=np.array(os_); ds_=np.array(ds_); tm=np.zeros(len(os_))
rs=oracle.ref_scene(sd)
h0=oracle.intersect("ref", rs, os_, ds_, tm, 0); h1=oracle.intersect("ref", rs, os_, ds_, tm, 1)
hp=oracle.intersect("port", oracle.port_scene(sd), os_, ds_, tm, 0)
for k in range(len(cells)):
    print(cells[k], 'ref bvh', int(h0[k,12]), h0[k,0], '| ref brute', int(h1[k,12]), h1[k,0], '| port', int(hp[k,12]), hp[k,0])
