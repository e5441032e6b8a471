"""CPU oracle for the span-query hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy fp64 (and hashlib) implementation of what the span-query
prefill path computes (§5.4-§5.6). It shares no code with the CUDA
path (`paper_2511_02749_b200/csrc`): no kernels, headers, helpers, tables or constants. The only
module both sides import is `paper_2511_02749_b200.inputs` (seeded input draws, no method
arithmetic).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import this package. The product path never does.

Modules
  rope       rotary encoding, rotate-half pairs (i, i+d/2), θ_i = base^(-2i/d)   [S:358, P:610]
  hashing    BLAKE2b-128 digest chains: prefix / fragment (suspended) / join fold / cross
             [P:97-98; SURVEY §8(c) hash contract]
  tree       ABI tree -> (prefix, fragments, cross) with ⊕ flattening           [P:205-251, P:439]
  store      content-hash block store + planner mirror (lookup, insert, alloc, LRU, pins)
             [P:94; SURVEY §8(c) R8-R13]
  attention  dense masked brute force (the plain definition) and the segment-wise form
             (fragments causal at span-local positions, join at global positions) [P:672]
  cidra      block repositioning (ReRoPE moves, chains, cycles, duplicates), the plain
             out-of-place definition                                          [P:610, P:618-627]

Parity status per function is listed in DESIGN.md §"Oracle pins"; every function here is pinned
by a `-m "not gpu"` test in tests/test_oracle_*.py except where its docstring says
"parity unpinned".
"""
