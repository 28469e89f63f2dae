"""B200-native world step of the non-episodic neuroevolution simulator (arXiv 2302.09334).

The product is libsim.so (paper_2302_09334_b200/csrc, C ABI in include/sim.h): hand-written
sm_100a kernels for regrowth, observation, per-agent LSTM policies, movement/physiology and
reproduction.  `sim` is its thin ctypes binding; `dist` holds the multi-process helpers.
"""
from .sim import World, SimError, lib, validate, state_sizes  # noqa: F401
