// blake2b.h — BLAKE2b (RFC 7693), unkeyed, variable digest length; used for the block
// digest chains of the span-query planner (§2, §5.4; DESIGN.md
// "Hash contract").
#pragma once
#include <cstddef>
#include <cstdint>

namespace spq {

// out <- BLAKE2b-(8*outlen)(data[0..len)), outlen in 1..64.
void blake2b(uint8_t* out, size_t outlen, const void* data, size_t len);
// Process-wide: use the scalar compression even where AVX2 is available (both produce the same
// digests; the switch lets tests check both paths).
void blake2b_force_scalar(bool on);

struct Digest {
  uint8_t b[16];
  bool operator==(const Digest& o) const;
};
struct DigestHash {
  size_t operator()(const Digest& d) const;
};

}  // namespace spq
