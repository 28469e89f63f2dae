"""Timeline of one k_policy_half launch (graph path) (diagnostic build with -DECO_POLICY_TRACE).

Per live agent the kernel records (start, mask ready, end, nnz) on the global timer; this
prints the distribution of those times relative to the first agent's start."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_09334_b200 import build as B  # noqa: E402

extra = tuple(d for d in os.environ.get("DIAG_DEFINES", "").split(",") if d)
diag = os.path.join(B.HERE, "libsim_trace.so")
if not (os.environ.get("DIAG_NOBUILD") and os.path.exists(diag)):
    B.build(defines=("ECO_POLICY_TRACE",) + extra, out=diag)
os.environ["ECO_LIBSIM_OVERRIDE"] = diag
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
flush = "--flush" in sys.argv  # L2 flushed before each traced step, as bench.py
world = sim.World(workloads.paper_scale(), device=0)
world.step(W)
world.synchronize()
if flush:
    import torch
    import bench
    fb = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    fr = torch.ones(bench.FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
for rep in range(3):
    world.phase_ns(reset=True)
    if flush:
        fb.zero_()
        fr.sum()
        torch.cuda.synchronize()
    world.step(1)
    world.synchronize()
    out = np.zeros(16 + 32768, np.int64)
    sim._check(sim.lib().sim_get_phase_ns(world._h, sim._ptr(out), -1))
    tr = out[16:].reshape(8192, 4)
    live = tr[:, 0] > 0
    t0 = tr[live, 0].min()
    st, mk, en, nnz = (tr[live, 0] - t0) / 1e3, (tr[live, 1] - t0) / 1e3, (tr[live, 2] - t0) / 1e3, tr[live, 3]
    if "ECO_POLICY_TRACE_STREAM" in extra:  # trace[3] holds the time the chunks were in
        sd = (tr[live, 3] - t0) / 1e3
        print(f"  stream done q50 {float(np.median(sd)):6.2f} (after mask {float(np.median(sd - mk)):6.2f}; "
              f"epilogue to end {float(np.median(en - sd)):6.2f}) us")
        nnz = np.zeros_like(nnz)
    n = int(live.sum())
    q = lambda a, f: float(np.quantile(a, f))
    print(f"step {world.t}: agents {n}, nnz mean {nnz.mean():.1f} max {nnz.max()}")
    print(f"  start  q50 {q(st, .5):6.2f} q90 {q(st, .9):6.2f} q99 {q(st, .99):6.2f} max {st.max():6.2f} us")
    print(f"  mask   q50 {q(mk, .5):6.2f} q90 {q(mk, .9):6.2f} max {mk.max():6.2f} (rel start q50 {q(mk - st, .5):6.2f})")
    print(f"  agent  (end - start) q50 {q(en - st, .5):6.2f} q90 {q(en - st, .9):6.2f} max {(en - st).max():6.2f}")
    print(f"  end    q50 {q(en, .5):6.2f} q90 {q(en, .9):6.2f} q99 {q(en, .99):6.2f} max {en.max():6.2f} us")
    late = st > q(st, .9)
    print(f"  agents starting after the first wave: {int((st > 2.0).sum())}")
    dur = en - st
    cc = np.corrcoef(nnz, dur)[0, 1]
    print(f"  corr(nnz, duration) {cc:.2f}; duration by nnz bucket:",
          {f"{lo}-{lo + 15}": round(float(dur[(nnz >= lo) & (nnz < lo + 16)].mean()), 2)
           for lo in range(0, 99, 16) if ((nnz >= lo) & (nnz < lo + 16)).any()})
