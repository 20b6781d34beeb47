import sys, numpy as np
sys.path.insert(0,'tests')
from conftest import load_golden, golden_scene
import paper_2303_11103_b200 as P
g = load_golden("canyon"); sc = golden_scene(g); b = P.build(sc)
ox, oy, cs, nx, ny, h, depth, nr = g["cov0_spec"]
grid = P.GridSpec((ox, oy), cs, int(nx), int(ny), h)
cm = P.coverage_map(sc, b, grid, int(depth), method=str(g["cov0_method"]), num_rays=int(nr))
want = g["cov0_gains"]
d = np.argwhere((cm.gains == 0) != (want == 0))
print("zero-pattern mismatches", len(d))
for iy, ix in d[:10]: print(iy, ix, cm.gains[iy, ix], want[iy, ix])
rel = np.abs(cm.gains - want) / np.maximum(want, 1e-300)
print("max rel", rel[want > 0].max())
# paths at one mismatching cell
if len(d):
    iy, ix = d[0]
    pt = grid.cell_center(ix, iy)
    tx = sc.devices[0]
    gain, paths = P.point_path_gain(sc, b, tx, pt, int(depth), "fibonacci", int(nr))
    print("ppg", gain, [(p.kind, p.seq) for p in paths])
    import oracle as O
    ob = O.Bvh(O.SceneArrays(sc))
    op = O.compute_paths_between(sc, ob, tx, P.probe_receiver(pt), int(depth), "fibonacci", int(nr))
    print("oracle", [(p.kind, p.seq) for p in op])
