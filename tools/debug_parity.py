"""Debug helper: detailed GPU-vs-oracle comparison on one config/view (prints mismatch stats)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import make_scene
from tests.gpu_common import gpu_scene

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
views = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [0]
sc = make_scene(cfg)
g = gpu_scene(sc, views)
img = g['R'].forward(g['atlas'], g['occ']).cpu().numpy()
planes, occ, _ = orc.pack(sc.levels)
print('pack equal', np.array_equal(g['atlas'].cpu().numpy(), planes))
for vi, v in enumerate(views):
    cam = sc.cameras[v]
    P = orc.project(planes, occ, cam)
    d = puv.debug_tensors(g['layout'], g['cams'], g['R'].state, g['R'].arena, vi)
    ref_depth = np.where(P['visible'] == 1, P['depth_bits'], np.uint32(0xFFFFFFFF)).astype(np.uint32)
    gd = d['depth_key'].cpu().numpy().view(np.uint32)
    print(f'view {v}: depth mismatches {(gd != ref_depth).sum()} nvis gpu {d["n_visible"]} ref {P["visible"].sum()}')
    order = d['depth_order'].cpu().numpy().view(np.uint32)
    vis = np.nonzero(P['visible'])[0]
    ref_order = vis[np.lexsort((vis, P['depth_bits'][vis]))]
    mm = np.nonzero(order != ref_order)[0]
    print('  depth order mismatches', mm.size, mm[:8], order[mm[:8]], ref_order[mm[:8]], 'dups', order.size - np.unique(order).size)
    start, end, gids = orc.binning(P, cam)
    ts = d['tile_start'].cpu().numpy().view(np.uint32); te = d['tile_end'].cpu().numpy().view(np.uint32)
    kg = d['keys_gid'].cpu().numpy().view(np.uint32)
    print(f'  K gpu {d["n_keys"]} ref {gids.size}; start mism {(ts != start).sum()} end mism {(te != end).sum()}')
    if kg.size == gids.size:
        mm = np.nonzero(kg != gids)[0]
        print(f'  list mismatches {mm.size}', mm[:10], kg[mm[:10]], gids[mm[:10]])
        if mm.size:
            t = np.searchsorted(end, mm[0], side='right'); print('  first bad tile', t, start[t], end[t])
            print('  gpu seg', kg[start[t]:end[t]][:40]); print('  ref seg', gids[start[t]:end[t]][:40])
    ref, T, nc, st = orc.forward(planes, occ, sc.sh_degree, cam)
    gT = d['t_final'].cpu().numpy(); gn = d['n_contrib'].cpu().numpy()
    print(f'  T mism {(gT.view(np.uint32) != T.view(np.uint32)).sum()} ncontrib mism {(gn != nc).sum()}')
    err = np.abs(img[vi] - ref)
    print(f'  img max err {err.max():.3e} n>1e-4 {(err.max(0) > 1e-4).sum()}')
    bad = np.argwhere(err.max(0) > 1e-4)[:5]
    for (j, i) in bad:
        print('   px', i, j, img[vi][:, j, i], ref[:, j, i], 'T', gT[j, i], T[j, i], 'nc', gn[j, i], nc[j, i])
    # which gids land in different tiles?
    from collections import defaultdict
    gt = defaultdict(set); rt = defaultdict(set)
    for t in range(len(start)):
        for x in kg[ts[t]:te[t]]: gt[int(x)].add(t)
        for x in gids[start[t]:end[t]]: rt[int(x)].add(t)
    diff = [x for x in set(gt) | set(rt) if gt[x] != rt[x]]
    print('  gids with different tile sets:', len(diff))
    gx = (cam.width + 15) // 16
    for x in diff[:6]:
        p = P[x]
        print('   gid', x, 'gpu tiles', sorted(gt[x])[:12], 'ref', sorted(rt[x])[:12], 'rect', p['x0'], p['x1'], p['y0'], p['y1'], 'mx', p['mx'], p['my'])
    # sorted-order check on the GPU lists (depth non-decreasing, gid tiebreak)
    bad_order = 0
    for t in range(len(start)):
        seg = kg[ts[t]:te[t]]
        dk = ref_depth[seg].astype(np.uint64) << 32 | seg.astype(np.uint64)
        bad_order += int((np.diff(dk.astype(np.int64)) <= 0).sum())
    print('  gpu lists out of order pairs:', bad_order)
