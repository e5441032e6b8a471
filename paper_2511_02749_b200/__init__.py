"""spanq-b200: B200-native span-query prefill (arXiv 2511.02749) behind a C ABI.

  include/spanq.h              the ABI (plan / lookup / insert / prefill_jobs / join / release)
  paper_2511_02749_b200/csrc   C++ planner + content-hash store, sm_100a CUDA kernels
  paper_2511_02749_b200/spanq  ctypes binding (marshalling only, no fallback)
  paper_2511_02749_b200/inputs seeded synthetic workloads (shared with the oracle)
"""
from . import inputs  # noqa: F401
