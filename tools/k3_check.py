"""Quick K3 (tcgen05 3xTF32) vs oracle check on configs 1-3 (+ config 4 antenna subset)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import workload  # noqa: E402
import paper_1802_05427_b200 as ce  # noqa: E402

kern = int(sys.argv[1]) if len(sys.argv) > 1 else ce.CE_KERNEL_TF32X3
for cfg_id, m_hi in ((1, None), (2, None), (3, None), (4, 8), (5, 4)):
    cfg = workload.get_config(cfg_id)
    r, s2 = workload.channel_stats(cfg, 0)
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x, m_hi=m_hi)
    soi = workload.set_of_instance(cfg)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=kern).build()
    t0 = time.time()
    h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda(),
                     set_of_instance=torch.from_numpy(soi).cuda())
    torch.cuda.synchronize()
    dt = time.time() - t0
    ref = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride)
    hn = h.cpu().numpy()
    err = oracle.rel_fro_error_per_instance(hn, ref)
    bad = np.argwhere(np.abs(hn - ref) > 1e-3 * np.abs(ref).max())
    print(f"config {cfg_id} kernel {kern}: max rel err {err.max():.3e}  finite {np.isfinite(hn).all()}  "
          f"first bad {bad[:3].tolist()}  {dt*1e3:.1f} ms", flush=True)
    est.close()
