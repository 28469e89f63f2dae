"""One world over several GPUs, agent-sharded (include/sim.h: sim_shard; SURVEY.md §8(e),
the agent-home variant of E.2).

Every rank (one process per GPU, torch.distributed over NCCL) holds the whole world and runs
its integer dynamics identically; slot s belongs to rank s % n_ranks (children inherit their
parent's rank) and only its owner runs that agent's policy from its own copy of the weights.
One step is

    sim_step_policy  ->  SUM-allreduce of the two exchange buffers  ->  sim_step_post

where the buffers are the move records by slot (zero for the other ranks' agents) and the
policy counters.  The allreduce is the step's only collective; everything runs on the
library's stream: the handle is created on torch's current stream of `device` when no
stream is given, and the allreduce is issued with that stream current, so NCCL (which
orders with torch's current stream) runs between sim_step_policy and sim_step_post.
The trajectory equals the unsharded world's exactly (tests/test_gpu_parity.py).
"""
from . import sim


def combine_(tensors, dist, group=None):
    """SUM-allreduce each tensor in place across the ranks (the exchange of one step)."""
    for t in tensors:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


class ShardedWorld:
    """A sim.World sharded over the ranks of an initialised torch.distributed group."""

    def __init__(self, wc, dist, device: int, stream=None, log_capacity: int = 0, group=None):
        self.dist, self.group = dist, group
        self.n_ranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        import torch
        if stream is None:  # the library must share NCCL's stream (torch's current one)
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.world = sim.World(wc, device=device, stream=stream, log_capacity=log_capacity)
        if self.n_ranks > 1:
            self.world.shard(self.n_ranks, self.rank)
            self._bufs = self.world.exchange_tensors()

    @property
    def t(self):
        return self.world.t

    def step(self, n: int = 1):
        if self.n_ranks == 1:
            self.world.step(n)
            return
        import torch
        with torch.cuda.stream(self.stream):
            for _ in range(n):
                self.world.step_policy()
                combine_(self._bufs, self.dist, self.group)
                self.world.step_post()

    def __getattr__(self, name):  # step_log, get_state, synchronize, destroy, ...
        return getattr(self.world, name)
