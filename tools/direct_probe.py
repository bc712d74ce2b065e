"""Trace one directional shadow ray of the direct golden case on the GPU and
on the host (same packed BVH); print the first divergence. Tools only."""
import ctypes as C
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _box(lo, hi, o, d, inv, tmax):
    tn, tf = 0.0, tmax
    for a in range(3):
        if d[a] == 0.0:
            if o[a] < lo[a] or o[a] > hi[a]:
                return False
        else:
            ta, tb = (lo[a] - o[a]) * inv[a], (hi[a] - o[a]) * inv[a]
            if ta > tb:
                ta, tb = tb, ta
            tn, tf = max(tn, ta) if ta > tn else tn, tb if tb < tf else tf
            if tn > tf:
                return False
    return tn <= tf


def _tri(r, o, d, tmax):
    v0, e1, e2 = r[0:3], r[3:6], r[6:9]
    pv = [d[1] * e2[2] - d[2] * e2[1], d[2] * e2[0] - d[0] * e2[2], d[0] * e2[1] - d[1] * e2[0]]
    det = e1[0] * pv[0] + e1[1] * pv[1] + e1[2] * pv[2]
    if abs(det) <= 1e-14:
        return False
    inv = 1.0 / det
    tv = [o[0] - v0[0], o[1] - v0[1], o[2] - v0[2]]
    u = (tv[0] * pv[0] + tv[1] * pv[1] + tv[2] * pv[2]) * inv
    if u < 0.0 or u > 1.0:
        return False
    qv = [tv[1] * e1[2] - tv[2] * e1[1], tv[2] * e1[0] - tv[0] * e1[2], tv[0] * e1[1] - tv[1] * e1[0]]
    v = (d[0] * qv[0] + d[1] * qv[1] + d[2] * qv[2]) * inv
    if v < 0.0 or u + v > 1.0:
        return False
    t = (e2[0] * qv[0] + e2[1] * qv[1] + e2[2] * qv[2]) * inv
    return t > 1e-9 and t < tmax


def host_log(nodes, tris, ray):
    o, d, tmax = [float(x) for x in ray[:3]], [float(x) for x in ray[3:6]], float(ray[6])
    inv = [0.0 if x == 0.0 else 1.0 / x for x in d]
    ints = nodes.view(np.int32)
    out, stack = [], [0]
    while stack:
        nd = stack.pop()
        h = _box(nodes[nd, :3].tolist(), nodes[nd, 3:6].tolist(), o, d, inv, tmax)
        out.append(nd if h else -1 - nd)
        if not h:
            continue
        l, r, st, cn = ints[nd, 12:16].tolist()
        if cn > 0:
            out += [(1000000 if _tri(tris[t].tolist(), o, d, tmax) else 2000000) + t
                    for t in range(st, st + cn)]
        else:
            stack += [r, l]
    return out


def main(i=172):
    from paper_2203_12339_b200.shadows import DirectionalLight, build_bvh
    so = ROOT / "tools" / "_direct_probe.so"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-shared", "-Xcompiler", "-fPIC", "-o", str(so),
                           str(ROOT / "tools" / "direct_probe.cu")])
    P = C.CDLL(str(so))
    g = dict(np.load(ROOT / "tests/golden/direct.npz"))
    bvh = build_bvh(g["positions"], g["triangles"])
    nodes, tris = bvh.packed()
    dl = DirectionalLight(direction=g["d_dir"], irradiance=g["d_irr"])
    p = g["positions"][i].astype(np.float32).astype(np.float64)
    n = g["normals"][i].astype(np.float32).astype(np.float64)
    o = p + bvh.ray_offset * n
    ray = np.concatenate([o, -dl.direction, [4.0 * bvh.bbox_diagonal + 1.0]])
    dn, dt, dr = (torch.as_tensor(a, device="cuda") for a in (nodes, tris, ray))
    log = torch.zeros(4096, dtype=torch.int32, device="cuda")
    rc = P.direct_probe(C.c_void_p(dn.data_ptr()), C.c_void_p(dt.data_ptr()), C.c_void_p(dr.data_ptr()),
                        C.c_void_p(log.data_ptr()), 4000)
    L = log.cpu().numpy().tolist()
    L = L[:L.index(-999999999)]
    print("rc", rc, "gpu log", L)
    print("ray", ray.tolist())
    H = host_log(nodes, tris, ray)
    print("host log", H)
    for k, (a, b) in enumerate(zip(L, H)):
        if a != b:
            print("first divergence at", k, a, b)
            break
    hits = [v - 1000000 for v in L if 1000000 <= v < 2000000]
    print("gpu triangle hits", hits)



def lib_check(i=172):
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.shadows import DirectionalLight, LightRig, build_bvh
    g = dict(np.load(ROOT / "tests/golden/direct.npz"))
    bvh = build_bvh(g["positions"], g["triangles"])
    nodes, tris = bvh.packed()
    rig = LightRig(lights=(DirectionalLight(direction=g["d_dir"], irradiance=g["d_irr"]),))
    d = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dt), device="cuda")
    for lo, hi in ((0, g["positions"].shape[0]), (i, i + 1)):
        pos, nrm = d(g["positions"][lo:hi], np.float32), d(g["normals"][lo:hi], np.float32)
        mat = d(np.array([1, 1, 1, 0.01, 0.01, 0.01, float(g["eta"])]), np.float64)
        E = torch.empty((3, hi - lo), dtype=torch.float64, device="cuda")
        kinds = torch.tensor(rig.kinds())
        keep = [d(rig.packed(), np.float64), d(nodes, np.float64), d(tris, np.float64)]
        _lib.call("sss_direct_irradiance", hi - lo, _lib.ptr(pos), _lib.ptr(nrm), 1, _lib.ptr(kinds),
                  _lib.ptr(keep[0]), _lib.ptr(mat), bvh.ray_offset, bvh.bbox_diagonal,
                  _lib.ptr(keep[1]), _lib.ptr(keep[2]), _lib.ptr(E), _lib.stream_ptr())
        torch.cuda.synchronize()
        print("lib", lo, hi, E[:, i - lo].tolist())


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
    lib_check(*[int(a) for a in sys.argv[1:]])
