// cidra.h — host planner of CIDRA block repositioning (§5.5.1).
//
// Input: moves i = (src[i] -> dst[i], delta[i]): block dst[i] must end up holding the ORIGINAL
// content of block src[i] with K re-encoded delta[i] positions later (ReRoPE) and V
// copied. A destination appears at most once; a source may feed several destinations (the
// paper's "duplication", which needs no scratch block here: the extra destinations are
// written from the source before the source itself is overwritten).
//
// Every node has at most one incoming move, so each connected component of the move graph is
// a tree (rooted at a block nobody writes) or one cycle with trees hanging off it ("the
// cycles and ... independent subgraphs"). The schedule lists, per component, moves in an order
// that is safe IN PLACE: a block is overwritten only after every move reading it has run
// (reverse BFS from the roots), and a cycle is rotated through one scratch slot (tmp <- last,
// c_i <- c_{i-1}, ..., c_0 <- tmp). Components are independent: the kernel runs them in parallel.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace spq {

// mode 0: dst <- R(src, delta); 1: tmp <- src (delta, dst unused); 2: dst <- R(tmp, delta)
struct CidraOp {
  int32_t dst, src, delta, mode;
};

struct CidraSchedule {
  std::vector<CidraOp> ops;
  std::vector<int32_t> comp_off;  // component c = ops[comp_off[c], comp_off[c+1])
  int64_t cycles = 0;             // components containing a cycle (one scratch slot each)
  int64_t duplicates = 0;         // sum over sources of max(0, out-degree - 1)
  int64_t max_component_ops = 0;
};

// false + *err on an out-of-range id or a destination written twice.
bool cidra_schedule(const int32_t* src, const int32_t* dst, const int32_t* delta, int64_t n, int64_t num_blocks,
                    CidraSchedule* out, std::string* err);

}  // namespace spq
