// blake2b.cpp — RFC 7693 BLAKE2b written from the RFC's algorithm description (§2-§3):
// 12 rounds of the G mixing function over a 16-word state, 128-byte blocks, 128-bit byte
// counter, final-block flag, parameter block {digest length, key length 0, fanout 1, depth 1}.
#include "blake2b.h"

#include <atomic>

#include <immintrin.h>

#include <cstdlib>
#include <cstring>

namespace spq {
namespace {

constexpr uint64_t kIV[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                             0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                             0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};

constexpr uint8_t kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

inline uint64_t load64(const uint8_t* p) {
  uint64_t v;
  std::memcpy(&v, p, 8);  // little-endian host (x86_64)
  return v;
}

#define SPQ_G(r, i, a, b, c, d)                 \
  do {                                          \
    v[a] = v[a] + v[b] + m[kSigma[r][2 * i]];     \
    v[d] = rotr(v[d] ^ v[a], 32);               \
    v[c] = v[c] + v[d];                         \
    v[b] = rotr(v[b] ^ v[c], 24);               \
    v[a] = v[a] + v[b] + m[kSigma[r][2 * i + 1]]; \
    v[d] = rotr(v[d] ^ v[a], 16);               \
    v[c] = v[c] + v[d];                         \
    v[b] = rotr(v[b] ^ v[c], 63);               \
  } while (0)
#define SPQ_ROUND(r)                 \
  do {                               \
    SPQ_G(r, 0, 0, 4, 8, 12);        \
    SPQ_G(r, 1, 1, 5, 9, 13);        \
    SPQ_G(r, 2, 2, 6, 10, 14);       \
    SPQ_G(r, 3, 3, 7, 11, 15);       \
    SPQ_G(r, 4, 0, 5, 10, 15);       \
    SPQ_G(r, 5, 1, 6, 11, 12);       \
    SPQ_G(r, 6, 2, 7, 8, 13);        \
    SPQ_G(r, 7, 3, 4, 9, 14);        \
  } while (0)

void compress(uint64_t* h, const uint8_t* block, uint64_t t_lo, uint64_t t_hi, bool last) {
  uint64_t m[16], v[16];
  for (int i = 0; i < 16; ++i) m[i] = load64(block + 8 * i);
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = kIV[i];
  }
  v[12] ^= t_lo;
  v[13] ^= t_hi;
  if (last) v[14] = ~v[14];
  // 12 rounds, fully unrolled with compile-time message schedule (RFC 7693 §3.2)
  SPQ_ROUND(0);
  SPQ_ROUND(1);
  SPQ_ROUND(2);
  SPQ_ROUND(3);
  SPQ_ROUND(4);
  SPQ_ROUND(5);
  SPQ_ROUND(6);
  SPQ_ROUND(7);
  SPQ_ROUND(8);
  SPQ_ROUND(9);
  SPQ_ROUND(10);
  SPQ_ROUND(11);
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}
#undef SPQ_ROUND
#undef SPQ_G

// The same compression with the 16-word state as four 256-bit rows (v0..3 | v4..7 | v8..11 |
// v12..15): the four column G's of a round run as one vector G, then the rows are rotated so the
// four diagonal G's do too (RFC 7693 §3.2's order of G applications, 4 at a time). Runtime
// dispatch: used only when the host CPU has AVX2 (the test suite checks both against hashlib).
__attribute__((target("avx2"))) inline __m256i rotr32(__m256i x) { return _mm256_shuffle_epi32(x, 0xB1); }
__attribute__((target("avx2"))) inline __m256i rotr24(__m256i x) {
  const __m256i r = _mm256_setr_epi8(3, 4, 5, 6, 7, 0, 1, 2, 11, 12, 13, 14, 15, 8, 9, 10, 3, 4, 5, 6, 7, 0, 1, 2, 11,
                                     12, 13, 14, 15, 8, 9, 10);
  return _mm256_shuffle_epi8(x, r);
}
__attribute__((target("avx2"))) inline __m256i rotr16(__m256i x) {
  const __m256i r = _mm256_setr_epi8(2, 3, 4, 5, 6, 7, 0, 1, 10, 11, 12, 13, 14, 15, 8, 9, 2, 3, 4, 5, 6, 7, 0, 1, 10,
                                     11, 12, 13, 14, 15, 8, 9);
  return _mm256_shuffle_epi8(x, r);
}
__attribute__((target("avx2"))) inline __m256i rotr63(__m256i x) {
  return _mm256_or_si256(_mm256_srli_epi64(x, 63), _mm256_add_epi64(x, x));
}

__attribute__((target("avx2"))) void compress_avx2(uint64_t* h, const uint8_t* block, uint64_t t_lo, uint64_t t_hi,
                                                   bool last) {
  uint64_t m[16];
  for (int i = 0; i < 16; ++i) m[i] = load64(block + 8 * i);
  const __m256i h0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(h));
  const __m256i h1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(h + 4));
  __m256i a = h0, b = h1;
  __m256i c = _mm256_setr_epi64x(static_cast<long long>(kIV[0]), static_cast<long long>(kIV[1]),
                                 static_cast<long long>(kIV[2]), static_cast<long long>(kIV[3]));
  __m256i d = _mm256_setr_epi64x(static_cast<long long>(kIV[4] ^ t_lo), static_cast<long long>(kIV[5] ^ t_hi),
                                 static_cast<long long>(last ? ~kIV[6] : kIV[6]), static_cast<long long>(kIV[7]));
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kSigma[r];
    // columns: G(i) for i = 0..3 on lanes i, message words s[2i], s[2i+1]
    __m256i x = _mm256_setr_epi64x(static_cast<long long>(m[s[0]]), static_cast<long long>(m[s[2]]),
                                   static_cast<long long>(m[s[4]]), static_cast<long long>(m[s[6]]));
    __m256i y = _mm256_setr_epi64x(static_cast<long long>(m[s[1]]), static_cast<long long>(m[s[3]]),
                                   static_cast<long long>(m[s[5]]), static_cast<long long>(m[s[7]]));
    a = _mm256_add_epi64(_mm256_add_epi64(a, b), x);
    d = rotr32(_mm256_xor_si256(d, a));
    c = _mm256_add_epi64(c, d);
    b = rotr24(_mm256_xor_si256(b, c));
    a = _mm256_add_epi64(_mm256_add_epi64(a, b), y);
    d = rotr16(_mm256_xor_si256(d, a));
    c = _mm256_add_epi64(c, d);
    b = rotr63(_mm256_xor_si256(b, c));
    // diagonals: lane j holds (v[j], v[4 + (j+1)%4], v[8 + (j+2)%4], v[12 + (j+3)%4])
    b = _mm256_permute4x64_epi64(b, _MM_SHUFFLE(0, 3, 2, 1));
    c = _mm256_permute4x64_epi64(c, _MM_SHUFFLE(1, 0, 3, 2));
    d = _mm256_permute4x64_epi64(d, _MM_SHUFFLE(2, 1, 0, 3));
    x = _mm256_setr_epi64x(static_cast<long long>(m[s[8]]), static_cast<long long>(m[s[10]]),
                           static_cast<long long>(m[s[12]]), static_cast<long long>(m[s[14]]));
    y = _mm256_setr_epi64x(static_cast<long long>(m[s[9]]), static_cast<long long>(m[s[11]]),
                           static_cast<long long>(m[s[13]]), static_cast<long long>(m[s[15]]));
    a = _mm256_add_epi64(_mm256_add_epi64(a, b), x);
    d = rotr32(_mm256_xor_si256(d, a));
    c = _mm256_add_epi64(c, d);
    b = rotr24(_mm256_xor_si256(b, c));
    a = _mm256_add_epi64(_mm256_add_epi64(a, b), y);
    d = rotr16(_mm256_xor_si256(d, a));
    c = _mm256_add_epi64(c, d);
    b = rotr63(_mm256_xor_si256(b, c));
    b = _mm256_permute4x64_epi64(b, _MM_SHUFFLE(2, 1, 0, 3));
    c = _mm256_permute4x64_epi64(c, _MM_SHUFFLE(1, 0, 3, 2));
    d = _mm256_permute4x64_epi64(d, _MM_SHUFFLE(0, 3, 2, 1));
  }
  _mm256_storeu_si256(reinterpret_cast<__m256i*>(h), _mm256_xor_si256(h0, _mm256_xor_si256(a, c)));
  _mm256_storeu_si256(reinterpret_cast<__m256i*>(h + 4), _mm256_xor_si256(h1, _mm256_xor_si256(b, d)));
}

using CompressFn = void (*)(uint64_t*, const uint8_t*, uint64_t, uint64_t, bool);
const bool kHaveAvx2 = __builtin_cpu_supports("avx2");
std::atomic<bool> g_force_scalar{false};  // SPQ_OPT_HASH_SCALAR (tests: both compressions)

}  // namespace

void blake2b_force_scalar(bool on) { g_force_scalar.store(on); }

void blake2b(uint8_t* out, size_t outlen, const void* data, size_t len) {
  uint64_t h[8];
  for (int i = 0; i < 8; ++i) h[i] = kIV[i];
  h[0] ^= 0x01010000ULL ^ static_cast<uint64_t>(outlen);  // fanout 1, depth 1, no key
  const uint8_t* p = static_cast<const uint8_t*>(data);
  uint64_t t = 0;
  const CompressFn kCompress = kHaveAvx2 && !g_force_scalar.load(std::memory_order_relaxed) ? compress_avx2 : compress;
  // all full blocks except the last one
  while (len > 128) {
    t += 128;
    kCompress(h, p, t, 0, false);
    p += 128;
    len -= 128;
  }
  uint8_t last[128] = {0};
  std::memcpy(last, p, len);
  t += len;
  kCompress(h, last, t, 0, true);
  uint8_t full[64];
  std::memcpy(full, h, 64);
  std::memcpy(out, full, outlen);
}

bool Digest::operator==(const Digest& o) const { return std::memcmp(b, o.b, 16) == 0; }

size_t DigestHash::operator()(const Digest& d) const {
  size_t v;
  std::memcpy(&v, d.b, sizeof(v));
  return v;
}

}  // namespace spq
