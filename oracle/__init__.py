"""CPU oracle for the SampleAttention hot path (TEST INFRASTRUCTURE ONLY).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline legs may
import this package.  The product package never does; a missing CUDA
extension is a hard error there, never a fallback to this code.
"""

from .blocksift_port import *  # noqa: F401,F403
