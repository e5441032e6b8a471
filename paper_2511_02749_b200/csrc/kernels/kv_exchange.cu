// kv_exchange.cu — K6: gather / scatter whole KV blocks of one layer between the paged pool and
// a packed exchange buffer (a join's remote fragment KV is gathered from the
// fragment's owner rank). The transfer itself is one NCCL all-to-all over NVLink issued by the
// binding; this kernel is the HBM side of it.
//
// Pool layout: K and V each [L][nblk][Hkv][bs][d], so one layer's block is a
// contiguous run of Hkv*bs*d elements. Buffer layout: [n][2 (K,V)][Hkv*bs*d] elements.
// HBM-bound copy: 16-byte vector loads/stores, consecutive threads on consecutive 16 B words
// (coalesced on both sides), grid = a multiple of the SM count with a grid-stride loop.
#include <algorithm>

#include "launch.h"

namespace spq {
namespace {

__global__ void __launch_bounds__(256) kv_exchange_kernel(const int32_t* __restrict__ blocks, int64_t n,
                                                          uint4* __restrict__ kpool, uint4* __restrict__ vpool,
                                                          uint4* __restrict__ buf, int64_t words_per_block,
                                                          int64_t layer_base_words, int scatter) {
  const int64_t total = n * 2 * words_per_block;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = w / (2 * words_per_block);
    const int64_t r = w - i * 2 * words_per_block;
    const int kv = r >= words_per_block;
    const int64_t off = r - kv * words_per_block;
    uint4* pool = kv ? vpool : kpool;
    uint4* p = pool + layer_base_words + static_cast<int64_t>(__ldg(blocks + i)) * words_per_block + off;
    if (scatter)
      *p = __ldcs(buf + w);
    else
      __stcs(buf + w, *p);
  }
}

}  // namespace

cudaError_t launch_kv_exchange(const KvExchangeArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int64_t block_bytes = static_cast<int64_t>(a.hkv) * a.bs * a.d * a.elt;
  if (block_bytes % 16 != 0) return cudaErrorInvalidValue;
  const int64_t wpb = block_bytes / 16;
  const int64_t layer_base = static_cast<int64_t>(a.layer) * a.nblk * wpb;
  const int64_t total = a.n * 2 * wpb;
  const int64_t want = (total + 255) / 256;
  const int grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(a.num_sms) * 8));
  kv_exchange_kernel<<<grid, 256, 0, st>>>(a.blocks, a.n, static_cast<uint4*>(a.k_pool), static_cast<uint4*>(a.v_pool),
                                           static_cast<uint4*>(a.buf), wpb, layer_base, a.scatter);
  return cudaGetLastError();
}

}  // namespace spq
