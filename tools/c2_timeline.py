import sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2203_12339_b200 import _lib
from paper_2203_12339_b200 import lighting as LT
from paper_2203_12339_b200.basis import OpticalMaterial, build_basis
from paper_2203_12339_b200.config import C2
from paper_2203_12339_b200.geometry import from_config
from paper_2203_12339_b200.precompute import precompute_compressed
from paper_2203_12339_b200.runtime import Scene, SHLight
_lib.load()
g = from_config(C2); b = build_basis(C2.K, C2.lattice)
dt = precompute_compressed(g, b, C2.levels, C2.step1_keep, C2.step2_fraction)
L0 = LT.random_sh_light(C2.sh_bands, 5)
m = OpticalMaterial(sigma_s_prime=C2.material[0], sigma_a=C2.material[1], eta=C2.material[2])
sc = Scene(g, dt, b, m, SHLight(L0))
for f in range(3): sc.set_light(SHLight(L0))
sc.capture()
for _ in range(5): sc.replay(False); sc.replay(True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(5):
        sc.replay(False); sc.replay(True); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = None
for e in evs[-14:]:
    if t0 is None: t0 = e.time_range.start
    print(e.name.split("(")[0][-40:], round(e.time_range.start - t0, 2), round(e.time_range.end - t0, 2))
print("kernel", sc.transfer_kernel)
