"""Where the host->device part of a cfg5 assemble goes: pageable (staged) against pinned inputs."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1806_07884_b200 import api, configs
cfg = configs.CONFIGS["cfg5"]
xy, h = configs.points("cfg5")
refs = configs.centres("cfg5")
k = api.KernelSpec(cfg.kernel, cfg.alpha)
pxy = torch.empty(xy.shape, dtype=torch.float64).pin_memory(); pxy.numpy()[:] = xy
ph = torch.empty(h.shape, dtype=torch.float64).pin_memory(); ph.numpy()[:] = h
with api.Engine(0) as e:
    e.set_centres(refs, k)
    e.assemble(xy, h); e.synchronize()   # centre-side setup out of the way
    for name, a, b in (("pageable", xy, h), ("pinned", pxy.numpy(), ph.numpy()), ("pageable", xy, h), ("pinned", pxy.numpy(), ph.numpy())):
        t = time.perf_counter(); e.assemble(a, b); e.synchronize(); dt = time.perf_counter() - t
        print(name, "assemble_ms %.1f" % (dt * 1e3), "-> %.1f GB/s incl. 57 ms of bin+K3" % (4.8 / dt), flush=True)
    d = torch.empty(xy.size + h.size, dtype=torch.float64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        d[:xy.size].copy_(pxy.view(-1), non_blocking=True); d[xy.size:].copy_(ph, non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print("pinned DMA only: %.1f ms = %.1f GB/s" % (dt * 1e3, 4.8 / dt), flush=True)
