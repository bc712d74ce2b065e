"""Design probe for a K-fused 'lanes own rows' transfer layout on the C3
operator: per ordering / chunking choice, the step count, lane utilisation,
term-plane load instructions and the L1 lines they touch.
Usage: python tools/kf_sim.py -> JSON lines."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pairs_of(dt):
    n, K = dt.n, dt.K
    dev = "cuda"
    rp = dt.rowptr.to(dev)
    cols = dt.cols.to(dev).long() & 0xffffffff
    lens = rp[:, 1:] - rp[:, :-1]
    k_of = torch.repeat_interleave(torch.arange(K, device=dev), lens.sum(1))
    row_of = torch.repeat_interleave(torch.arange(n, device=dev).repeat(K), lens.reshape(-1))
    key = row_of * n + cols
    uk, inv = torch.unique(key, return_inverse=True)
    mask = torch.zeros(uk.numel(), dtype=torch.long, device=dev)
    mask.scatter_add_(0, inv, torch.bitwise_left_shift(torch.ones_like(k_of), k_of))
    return uk // n, uk % n, mask


def popc8(m):
    c = torch.zeros_like(m)
    for k in range(8):
        c += (m >> k) & 1
    return c


def sim(prow, pcol, mask, n, chunk, order, T2, group_by="class_len"):
    dev = prow.device
    npair = prow.numel()
    # row chunks of <= chunk pairs
    cnt = torch.bincount(prow, minlength=n)
    start = torch.cumsum(cnt, 0) - cnt
    pos = torch.arange(npair, device=dev) - start[prow]  # pairs are row-major, col-sorted
    # ordering inside a row
    pc = popc8(mask)
    if order == "col":
        okey = pos
    elif order == "mask":
        okey = (255 - mask) * 65536 + pcol
    elif order == "popc_mask":
        okey = ((8 - pc) * 256 + (255 - mask)) * 65536 + pcol
    elif order == "hi_mask":  # masks ordered by highest term first
        rev = torch.zeros_like(mask)
        for k in range(8):
            rev |= ((mask >> k) & 1) << (7 - k)
        okey = rev * 65536 + pcol
    else:
        raise ValueError(order)
    o = torch.argsort(prow * (1 << 40) + okey)
    prow, pcol, mask, pc = prow[o], pcol[o], mask[o], pc[o]
    pos = torch.arange(npair, device=dev) - start[prow]
    chunk_id_in_row = pos // chunk
    nch_row = (cnt + chunk - 1) // chunk
    ch_base = torch.cumsum(nch_row, 0) - nch_row
    cid = ch_base[prow] + chunk_id_in_row
    nchunks = int(nch_row.sum())
    clen = torch.bincount(cid, minlength=nchunks)
    crow = torch.repeat_interleave(torch.arange(n, device=dev), nch_row)
    local = crow % T2
    lvl = torch.zeros_like(local)
    for L in range(1, 4):
        lvl[(local >= 4 ** (L - 1)) & (local < 4 ** L)] = L
    if group_by == "class_len":
        gkey = lvl * (1 << 40) + (1 << 30) - clen
    elif group_by == "local_tile":
        gkey = local * (1 << 30) + crow // T2
    else:
        gkey = (1 << 30) - clen
    corder = torch.argsort(gkey)
    rank = torch.empty_like(corder)
    rank[corder] = torch.arange(nchunks, device=dev)
    warp = rank[cid] // 32
    lane = rank[cid] % 32
    s = pos % chunk
    nw = (nchunks + 31) // 32
    # steps per warp = max chunk length in the warp
    wlen = torch.zeros(nw, dtype=torch.long, device=dev).scatter_reduce_(
        0, torch.arange(nchunks, device=dev) // 32, clen[corder], "amax")
    steps = int(wlen.sum())
    sbase = torch.cumsum(wlen, 0) - wlen
    sid = sbase[warp] + s
    # per step: b_k and M
    bk = torch.zeros((steps, 8), dtype=torch.long, device=dev)
    for k in range(8):
        sel = ((mask >> k) & 1).bool()
        bk[:, k].index_add_(0, sid[sel], torch.bitwise_left_shift(torch.ones_like(lane[sel]), lane[sel]))
    nz = bk != 0
    plane_instr = int(nz.sum())
    pk = torch.zeros_like(bk)
    for b in range(32):
        pk += (bk >> b) & 1
    # value offsets: planes contiguous in (step, k) order
    m = pk.reshape(-1)
    off = torch.cumsum(m, 0) - m
    valid = m > 0
    first = (off[valid] * 4) // 128
    last = ((off[valid] + m[valid] - 1) * 4) // 128
    plane_lines = int((last - first + 1).sum())
    bs = torch.zeros(steps, dtype=torch.long, device=dev).index_add_(
        0, sid, torch.ones_like(sid))
    out = {"chunk": chunk, "order": order, "group": group_by, "pairs": npair, "chunks": nchunks,
           "warps": nw, "steps": steps, "lane_util": round(npair / (32 * steps), 4),
           "plane_instr": plane_instr, "plane_instr_per_step": round(plane_instr / steps, 3),
           "plane_eff": round(float(m.sum()) / (32 * plane_instr), 4),
           "plane_lines": plane_lines, "plane_lines_per_step": round(plane_lines / steps, 3),
           "multi_chunk_rows": int((nch_row > 1).sum()), "partials": int(nch_row[nch_row > 1].sum()),
           "max_warp_steps": int(wlen.max()), "mean_active_lanes": round(float(bs.float().mean()), 2)}
    return out


def main():
    import bench as B
    from paper_2203_12339_b200 import _lib
    from paper_2203_12339_b200.config import CONFIGS

    _lib.load()
    cfg = CONFIGS["env_large_256"]
    g, b, dt, env, sc = B.setup_scene(cfg, 0, torch, {})
    prow, pcol, mask = pairs_of(dt)
    T2 = (1 << dt.levels) ** 2
    pc = popc8(mask)
    # fill by row class
    local = prow % T2
    lvl = torch.zeros_like(local)
    for L in range(1, 4):
        lvl[(local >= 4 ** (L - 1)) & (local < 4 ** L)] = L
    print(json.dumps({"fill_by_row_class": [round(float(pc[lvl == L].float().mean()), 3) for L in range(4)],
                      "pairs_by_row_class": [int((lvl == L).sum()) for L in range(4)],
                      "mask_top": torch.bincount(mask, minlength=256).topk(12).indices.tolist(),
                      "mask_top_counts": torch.bincount(mask, minlength=256).topk(12).values.tolist()}),
          flush=True)
    for chunk in (256, 512):
        for order in ("col", "mask", "popc_mask", "hi_mask"):
            for gb in ("class_len", "local_tile"):
                print(json.dumps(sim(prow, pcol, mask, dt.n, chunk, order, T2, gb)), flush=True)


if __name__ == "__main__":
    main()
