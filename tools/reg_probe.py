import time, numpy as np, torch, ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
import torch.cuda
rt = torch.cuda.cudart()
B=1<<20
for nb in (8<<20, 48<<20, 168<<20):
    a = np.random.default_rng(0).random(nb//8)
    ts=[]
    for _ in range(3):
        t0=time.perf_counter(); r=rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0); t1=time.perf_counter()
        rt.cudaHostUnregister(a.ctypes.data); t2=time.perf_counter()
        ts.append(((t1-t0)*1e3,(t2-t1)*1e3, int(r)))
    print(nb>>20, "MiB register/unregister ms", ts)
print(torch.cuda.get_device_properties(0))
import subprocess
