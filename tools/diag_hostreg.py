import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
a = ds.data
cr = torch.cuda.cudart()
dev = torch.device('cuda', 0)
buf = torch.empty(a.size, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    buf.copy_(torch.from_numpy(a.reshape(-1)), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms (rc {rc}), H2D {1e3*(t2-t1):.1f} ms, unregister {1e3*(t3-t2):.1f} ms")
from paper_2212_10733_b200 import hostio
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hostio.upload_planes(a, dev); torch.cuda.synchronize()
    print(f"staged upload {1e3*(time.perf_counter()-t0):.1f} ms")
# bytes alloc with/without hugepage advice
import ctypes
for huge in (False, True):
    for rep in range(2):
        t0 = time.perf_counter()
        src = torch.empty(220_000_000, dtype=torch.uint8, device=dev)
        b = hostio.download_bytes(src, 220_000_000, b"x" * 13000) if not huge else None
        if huge:
            b = hostio.download_bytes(src, 220_000_000, b"x" * 13000)
        print('download_bytes', huge, f"{1e3*(time.perf_counter()-t0):.1f} ms")
        del b
