"""Per-block k_post phase clocks (diagnostic build with -DECO_BLOCK_CLOCK).

Builds libsim_diag.so, runs the paper-scale world for W + K steps and prints, per phase,
the distribution over blocks of own work and barrier wait (us per step)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_09334_b200 import build as B  # noqa: E402

extra = tuple(d for d in os.environ.get("DIAG_DEFINES", "").split(",") if d)
tag = "_".join(x.replace("=", "") for x in extra)
diag = os.path.join(B.HERE, f"libsim_diag{tag}.so")
if not (os.environ.get("DIAG_NOBUILD") and os.path.exists(diag)):
    B.build(defines=("ECO_BLOCK_CLOCK",) + extra, out=diag)
print("defines", extra)
os.environ["ECO_LIBSIM_OVERRIDE"] = diag
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W, K = int(sys.argv[1]) if len(sys.argv) > 1 else 2000, int(sys.argv[2]) if len(sys.argv) > 2 else 1000
world = sim.World(workloads.paper_scale(), device=0)
world.step(W)
world.synchronize()
world.phase_ns(reset=True)
world.step(K)
world.synchronize()
out = np.zeros(16 + 32768, np.int64)
sim._check(sim.lib().sim_get_phase_ns(world._h, sim._ptr(out), -1))
nb = 148
blk = out[16:16 + 4 * nb * 3].reshape(4, nb, 3) / K / 1e3
names = ("move", "claim", "1w:regrow|flag|end", "tail")
for k in range(4):
    wk, wt, fn = blk[k, :, 0], blk[k, :, 1], blk[k, :, 2]
    order = np.argsort(-wk)[:5]
    print(f"{names[k]:14s} work: min {wk.min():6.2f} med {np.median(wk):6.2f} max {wk.max():6.2f} (blocks {order.tolist()})"
          f"  wait: min {wt.min():6.2f} med {np.median(wt):6.2f} max {wt.max():6.2f}"
          f"  fence: min {fn.min():6.2f} med {np.median(fn):6.2f} max {fn.max():6.2f}")
print("regrow warps: cycles/warp", out[10] / max(out[12], 1) / K * K, "ns/warp", out[11] / max(out[12], 1), "warps/step", out[12] / K)
print("block0 phases", {k: v / K / 1e3 for k, v in zip(sim.POST_PHASES, out[:len(sim.POST_PHASES)])})
