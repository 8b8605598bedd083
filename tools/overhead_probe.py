import time, numpy as np, sys
sys.path.insert(0,'.')
from paper_2006_04391_b200 import _lib, homogenize as H
from paper_2006_04391_b200.evaluator import StrategyConfig
cfg=StrategyConfig(strategy="automatic", integrator="implicit-euler")
for n in (32, 64, 128, 256):
    grid=H.toy_mmc_grid(n); hom=H.Homogenizer(grid,cfg); lib=_lib.load()
    path=H.LoadingPath(steps=20); t=path.times(); eb=np.zeros(6); eb[0]=path.eps_xx(t)[1]
    free=np.array([False]+[True]*5)
    hom._solve(eb, t[1]-t[0], free)  # warm
    hom2=H.Homogenizer(grid,cfg)
    _lib.check(lib.am_solver_timing(hom2._h,1,None))
    t0=time.perf_counter(); info,_=hom2._solve(eb, t[1]-t[0], free); wall=time.perf_counter()-t0
    ph=np.zeros(5); _lib.check(lib.am_solver_timing(hom2._h,-1,_lib.ptr(ph)))
    k=ph[4]; dev=(ph[0]+ph[1]+ph[2]+ph[3])/k
    hom3=H.Homogenizer(grid,cfg)
    t0=time.perf_counter(); info,_=hom3._solve(eb, t[1]-t[0], free); wall3=time.perf_counter()-t0
    print(n, info.iterations, 'wall/it ms (timing on)', round(wall/info.iterations*1e3,3), 'wall/it (timing off)', round(wall3/info.iterations*1e3,3), 'device/it', round(dev,3), [round(x/k,3) for x in ph[:4]], flush=True)
