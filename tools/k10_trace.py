"""K10 per-CTA event trace (build libce with CE_NVCC_EXTRA=-DCE_K10_TRACE): where a unit's time goes.

Slots per CTA (clock64, SM clock): 0 start, 1 epilogue end; per unit i < 40: 8+i producer issued the LS tile,
168+i MMA issuer begins waiting, 208+i tmem_empty passed, 48+i b_full passed (MMAs issue), 88+i epilogue got
tmem_full, 128+i epilogue (warp 2) done with the unit."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1802_05427_b200 as ce  # noqa: E402
import workload  # noqa: E402

cfg = workload.get_comb_config("massive_12w")
r, s2 = workload.comb_stats(cfg)
x = workload.comb_pilots(cfg)
y = workload.comb_instances(cfg, x=x)
est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
yd, xd = torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda()
out = est.estimate(yd, xd)
for _ in range(3):
    est.estimate(yd, xd, out=out)
torch.cuda.synchronize()
tr = torch.zeros(148 * 1024, dtype=torch.int64, device="cuda")
lib = ce.ce.lib
lib.ce_k10_trace_set.argtypes = [ctypes.c_void_p]
lib.ce_k10_trace_set(ctypes.c_void_p(tr.data_ptr()))
est.estimate(yd, xd, out=out)
torch.cuda.synchronize()
lib.ce_k10_trace_set(ctypes.c_void_p(0))
t = tr.cpu().numpy().reshape(148, 1024).astype(np.float64)
t0 = t[:, 0:1]
rel = (t - t0) / 1.9e3   # us at ~1.9 GHz
print("CTA total (us): median %.1f max %.1f" % (np.median(rel[:, 1]), rel[:, 1].max()))
for c in (0, 50, 147):
    print("CTA", c)
    for i in range(0, 38, 3):
        print("  unit %2d  P %6.2f  Mwait %6.2f  Mtmem %6.2f  Mgo %6.2f  Efull %6.2f  Edone %6.2f" % (
            i, rel[c, 8 + i], rel[c, 168 + i], rel[c, 208 + i], rel[c, 48 + i], rel[c, 88 + i], rel[c, 128 + i]))
d_full = rel[:, 88 + 1:88 + 38] - rel[:, 88:88 + 37]
print("epilogue unit period (us): median %.3f" % np.median(d_full))
print("MMA wait for b_full after tmem_empty (us): median %.3f" % np.median(rel[:, 48:48 + 38] - rel[:, 208:208 + 38]))
print("MMA wait for tmem_empty (us): median %.3f" % np.median(rel[:, 208:208 + 38] - rel[:, 168:168 + 38]))
print("epilogue busy per unit (us): median %.3f" % np.median(rel[:, 128:128 + 38] - rel[:, 88:88 + 38]))

m = lambda a, b: np.median(rel[:, b:b + 38] - rel[:, a:a + 38])
print("epilogue: tmem_full -> loads done %.3f; -> blk0 wait_read done %.3f; blk0 STS %.3f; blk0 fence %.3f; "
      "blk0 fence -> blk1 wait_read done %.3f; blk1 STS %.3f; blk1 fence %.3f; blk1 -> unit done %.3f" % (
          m(88, 256), m(256, 296), m(296, 376), m(376, 456), m(456, 336), m(336, 416), m(416, 496), m(496, 128)))
