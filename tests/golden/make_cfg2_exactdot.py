"""Generate tests/golden/cfg2_oracle_exactdot.json: the cfg2 two-scale PCG
(52^3, N=7, tol 1e-8) computed by the oracle restatement with its dot
products correctly rounded (orc_set_dot_mode(1)) instead of the reference's
sequential summation (krylov.cpp:11-16). Everything else in the oracle is
the reference's arithmetic, so the difference between this history and the
reference's golden (cfg2_pcg.json) is the reference's own dot-product
rounding: the floor any re-implementation is judged against.
Takes ~25 min on one core: python tests/golden/make_cfg2_exactdot.py"""
import sys, json, time, ctypes as C, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import OracleSystem, RefConfig
from oracle.ctypes_oracle import _ORC_SO, _load
L=_load(_ORC_SO,'orc_'); L.orc_set_dot_mode.argtypes=[C.c_int]; L.orc_set_dot_mode.restype=None
t=time.time()
s=OracleSystem(RefConfig(k=52,order=7,precond='two_scale'))
print('setup',time.time()-t, flush=True)
b=s.load_ones()
out={}
for mode in (1,):
    L.orc_set_dot_mode(mode)
    t=time.time()
    r=s.pcg(b,tol=1e-8,max_iterations=100)
    out[mode]={'iterations':r['iterations'],'residual_history':r['residual_history'].tolist(),'u_norm2':float(np.linalg.norm(r['u'])),'s':time.time()-t}
    print(mode, r['iterations'], time.time()-t, flush=True)
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'cfg2_oracle_exactdot.json'), 'w'))
