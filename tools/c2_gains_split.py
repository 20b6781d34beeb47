import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2303_11103_b200 as P
from paper_2303_11103_b200 import scenes, em
from paper_2303_11103_b200 import _native as N
from paper_2303_11103_b200.scene import element_layout
sc = scenes.street_canyon(n_per_row=100)
bvh = P.build(sc)
ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
for _ in range(5): P.build_cir(P.compute_gains(sc, bvh, ps))
torch.cuda.synchronize()
acc = {}
def mark(name, t0):
    t = time.perf_counter(); acc[name] = acc.get(name, 0) + t - t0; return t
R = 50
for _ in range(R):
    t = time.perf_counter()
    ctx = em.EvalContext(sc); T = ps.table; lam = sc.wavelength
    off_tx, sl_tx = element_layout(sc.tx_array, lam); off_rx, sl_rx = element_layout(sc.rx_array, lam)
    t = mark("layout", t)
    devs = {d.name: d for d in sc.devices}
    txr = ctx.rotation_rows_many([devs[n] for n in T.tx_names]); rxr = ctx.rotation_rows_many([devs[n] for n in T.rx_names])
    t = mark("rows", t)
    rows_t = em._rows_array(txr); rows_r = em._rows_array(rxr)
    otw = np.einsum("ek,dmk->dem", np.asarray(off_tx, dtype=np.float64), rows_t); orw = np.einsum("ek,dmk->dem", np.asarray(off_rx, dtype=np.float64), rows_r)
    eta_host = ctx.eta_values(bvh)
    t = mark("numpy prep", t)
    g = P.compute_gains(sc, bvh, ps)
    t = mark("compute_gains total", t)
    em._fraunhofer_warnings(sc, T, off_tx, off_rx, txr, rxr)
    t = mark("fraunhofer", t)
    c = P.build_cir(g)
    t = mark("build_cir", t)
torch.cuda.synchronize()
for k, v in acc.items(): print(f"{k:22s} {1e6*v/R:8.1f} us")
