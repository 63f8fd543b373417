"""GPU check of the binning pipeline against numpy on random screen arrays."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_18334_b200.engine import Engine, grid_dims

for n, W, H, seed in ((50, 64, 48, 0), (3000, 160, 96, 1), (200000, 1920, 1080, 2)):
    rng = np.random.default_rng(seed)
    mean2d = np.stack([rng.uniform(-20, W + 20, n), rng.uniform(-20, H + 20, n)], 1)
    radius = rng.uniform(0.5, 40, n)
    depth = rng.choice(np.linspace(1, 5, max(n // 3, 2)), n)   # many ties
    valid = rng.uniform(0, 1, n) < 0.95
    eng = Engine()
    dev = eng.device
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
    m = eng.bin_arrays(t(mean2d, np.float64), t(radius, np.float64), t(depth, np.float64),
                       t(valid, np.uint8), W, H)
    ntx, nty = grid_dims(W, H)
    ip, it, rg = eng.grid(ntx * nty)
    ip = ip.cpu().numpy().astype(np.int64)
    it = it.cpu().numpy().astype(np.int64) & 0xFFFF
    rg = rg.cpu().numpy().astype(np.int64)
    # numpy reference (tiles.py:43-79)
    r = np.ceil(radius)
    x0 = np.clip(np.floor((mean2d[:, 0] - r) / 16), 0, ntx).astype(np.int64)
    x1 = np.clip(np.floor((mean2d[:, 0] + r) / 16) + 1, 0, ntx).astype(np.int64)
    y0 = np.clip(np.floor((mean2d[:, 1] - r) / 16), 0, nty).astype(np.int64)
    y1 = np.clip(np.floor((mean2d[:, 1] + r) / 16) + 1, 0, nty).astype(np.int64)
    nx = np.where(valid, x1 - x0, 0).clip(min=0)
    ny = np.where(valid, y1 - y0, 0).clip(min=0)
    counts = nx * ny
    prim = np.repeat(np.arange(n), counts)
    off = np.concatenate([[0], np.cumsum(counts)[:-1]])
    within = np.arange(counts.sum()) - np.repeat(off, counts)
    nxr = np.repeat(nx, counts)
    tile = (np.repeat(y0, counts) + within // nxr) * ntx + np.repeat(x0, counts) + within % nxr
    dord = eng.depth_order[:n].cpu().numpy().astype(np.int64)
    roff = eng.rank_offset[:n + 1].cpu().numpy()
    keyd = np.where(counts > 0, depth, np.inf)
    want_ord = np.argsort(keyd, kind="stable")
    cz = counts[dord]
    print("  depth order ok (valid part):", np.array_equal(dord[counts[dord] > 0], want_ord[counts[want_ord] > 0]),
          " rank_offset ok:", np.array_equal(roff, np.concatenate([[0], np.cumsum(cz)])))
    order = np.lexsort((prim, depth[prim], tile))
    want_p, want_t = prim[order], tile[order]
    starts = np.searchsorted(want_t, np.arange(ntx * nty), "left")
    ends = np.searchsorted(want_t, np.arange(ntx * nty), "right")
    ok_m = m == len(want_p)
    print(f"n={n} M={m} want={len(want_p)} prim_eq={ok_m and np.array_equal(ip, want_p)} "
          f"tile_eq={ok_m and np.array_equal(it, want_t)} "
          f"ranges_eq={np.array_equal(rg[:, 0], starts) and np.array_equal(rg[:, 1], ends)}")
    if ok_m and not np.array_equal(it, want_t):
        bad = np.nonzero(it != want_t)[0]
        print("  first bad tile idx", bad[:5], it[bad[:5]], want_t[bad[:5]])
    if ok_m and not np.array_equal(ip, want_p):
        bad = np.nonzero(ip != want_p)[0]
        print("  first bad prim idx", bad[:5], ip[bad[:5]], want_p[bad[:5]], "n bad", len(bad))
