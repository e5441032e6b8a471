// tc2_rate.cu — issue-rate microbenchmark of the CTA-pair (cta_group::2) MMA forms, next to the
// single-CTA ones (tools/tc_rate.cu): clusters of 2, the leader issues M = 256 MMAs.
//   mode 0: SS N=64  (B split: 32 rows per CTA)   8 x K16 per group
//   mode 1: SS N=128 (64 rows per CTA)
//   mode 2: SS N=256 (128 rows per CTA)
//   mode 3: TS N=128 (A from TMEM, B MN-major: 64 columns per CTA)
//   mode 4: one paired-kernel step: 2 x (8 SS N64) + 2 x (4 TS N128)
//   mode 5: the same step with 128-key S tiles: 2 x (8 SS N128) + 2 x (8 TS N128) per 128 keys
//   mode 6: mode 4 with the two chains issued by two threads (warps 0 and 1 of the leader)
//   mode 7: mode 6 + the kernel's per-step commits (multicast, two per MMA group)
//   mode 8: mode 7 + before each group a wait (acquire.cluster) on a completed barrier and
//           tcgen05.fence::after_thread_sync, as the kernel's operand waits do
//   mode 9: mode 8 with CTA-scope waits (no .cluster)
//   mode 10: cross-CTA ping-pong: leader arrives on the peer's barrier, the peer waits and arrives
//            back on the leader's (remote arrive + acquire.cluster waits), cycles per round trip
//   mode 11: the kernel's step signal: leader issues one M=256 MMA + multicast commit, the peer
//            waits its copy and arrives on the leader's barrier, the leader waits: per round trip
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc2_rate.cu -o tools/tc2_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2511_02749_b200/csrc/kernels/sm100.cuh"

using namespace spq;

struct Sm {
  alignas(1024) uint8_t a[32768];
  alignas(1024) uint8_t b[32768];
  uint64_t bar, bar2, done, dummy[4], ping, pong;
  uint32_t tmem;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) rate2(int mode, int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  Sm& s = *reinterpret_cast<Sm*>(raw);
  const int t = threadIdx.x, warp = t / 32;
  const uint32_t rank = cluster_rank();
  for (int i = t; i < 32768 / 4; i += 128) {
    reinterpret_cast<uint32_t*>(s.a)[i] = 0x3c003c00u;
    reinterpret_cast<uint32_t*>(s.b)[i] = 0x3c003c00u;
  }
  if (t == 0) {
    mbar_init(&s.bar, 1);
    mbar_init(&s.bar2, 1);
    mbar_init(&s.done, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&s.dummy[i], 1 << 20);
    mbar_init(&s.ping, 1);
    mbar_init(&s.pong, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc2<512>(&s.tmem);
  if (t == 0) mbar_arrive(&s.done);  // phase 0 of `done` completes: later waits return at once
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = s.tmem;
  long long t0 = clock64();
  if (mode >= 10) {
    if (t == 0) {
      for (int it = 0; it < iters; ++it) {
        if (rank == 0) {
          if (mode == 10) {
            mbar_arrive_cl(cluster_addr(&s.ping, 1));
          } else {
            mma2_ss(tm, desc_sw128(smem_u32(s.a), 16, 1024), desc_sw128(smem_u32(s.b), 16, 1024),
                    idesc_bf16_f32(256, 64, false, false), 1u);
            mma_commit2(&s.ping);
          }
          mbar_wait_cl(&s.pong, it & 1);
        } else {
          mbar_wait_cl(&s.ping, it & 1);
          mbar_arrive_cl(cluster_addr(&s.pong, 0));
        }
      }
      if (mode == 11 && rank == 0) mbar_wait_cl(&s.ping, iters & 1 ? 0 : 1);  // own copy of the last commit
    }
  } else if (mode >= 6 && rank == 0 && (t == 0 || t == 32)) {
    const uint32_t a = smem_u32(s.a), b = smem_u32(s.b);
    const int x = t / 32;
    const uint32_t idS = idesc_bf16_f32(256, 64, false, false);
    const uint32_t idO = idesc_bf16_f32(256, 128, false, true);
    for (int it = 0; it < iters; ++it) {
      if (mode == 8) { mbar_wait_cl(&s.done, 0); tc_fence_after(); }
      if (mode == 9) { mbar_wait(&s.done, 0); tc_fence_after(); }
      for (int kk = 0; kk < 8; ++kk)
        mma2_ss(tm + 64 * x, desc_sw128(a + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                desc_sw128(b + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idS, 1u);
      if (mode >= 7) { mma_commit2(&s.dummy[0]); mma_commit2(&s.dummy[1]); }
      if (mode == 8) { mbar_wait_cl(&s.done, 0); tc_fence_after(); }
      if (mode == 9) { mbar_wait(&s.done, 0); tc_fence_after(); }
      for (int kk = 0; kk < 4; ++kk)
        mma2_ts(tm + 256 + 128 * x, tm + 128 + kk * 8, desc_sw128(b + kk * 2048, 8192, 1024), idO, 1u);
      if (mode >= 7) { mma_commit2(&s.dummy[2]); mma_commit2(&s.dummy[3]); }
    }
    mma_commit2(x == 0 ? &s.bar : &s.bar2);
  } else if (mode < 6 && rank == 0 && t == 0) {
    const uint32_t a = smem_u32(s.a), b = smem_u32(s.b);
    const int n = mode == 0 ? 64 : mode == 1 ? 128 : 256;
    for (int it = 0; it < iters; ++it) {
      if (mode <= 2) {
        const uint32_t id = idesc_bf16_f32(256, n, false, false);
        for (int kk = 0; kk < 8; ++kk)
          mma2_ss(tm, desc_sw128(a + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                  desc_sw128(b + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024), id, 1u);
      } else if (mode == 3) {
        const uint32_t id = idesc_bf16_f32(256, 128, false, true);
        for (int kk = 0; kk < 8; ++kk)
          mma2_ts(tm + 256, tm + 128 + kk * 8, desc_sw128(b + kk * 2048, 8192, 1024), id, 1u);
      } else {
        const int ns = mode == 4 ? 64 : 128;
        const uint32_t idS = idesc_bf16_f32(256, ns, false, false);
        const uint32_t idO = idesc_bf16_f32(256, 128, false, true);
        for (int x = 0; x < 2; ++x)
          for (int kk = 0; kk < 8; ++kk)
            mma2_ss(tm + 64 * x, desc_sw128(a + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                    desc_sw128(b + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idS, 1u);
        for (int x = 0; x < 2; ++x)
          for (int kk = 0; kk < ns / 16; ++kk)
            mma2_ts(tm + 256 + 128 * x, tm + 128 + (kk % 4) * 8, desc_sw128(b + kk * 2048, 8192, 1024), idO, 1u);
      }
    }
    mma_commit2(&s.bar);
  }
  if (mode < 10) mbar_wait(&s.bar, 0);
  if (mode >= 6 && mode < 10) mbar_wait(&s.bar2, 0);
  long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc2<512>(tm);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = sizeof(Sm);
  cudaFuncSetAttribute(rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"pair SS N64 (8 x 256x64x16)", "pair SS N128 (8 x 256x128x16)", "pair SS N256 (8 x 256x256x16)",
                         "pair TS N128 (8 x 256x128x16)", "pair step 64 keys: 2x8 SS N64 + 2x4 TS",
                         "pair step 128 keys: 2x8 SS N128 + 2x8 TS", "pair step 64 keys, 2 issuing threads",
                         "  + commits", "  + acquire.cluster waits + fence::after", "  + CTA-scope waits + fence::after",
                         "cross-CTA remote-arrive ping-pong", "MMA commit2 -> peer -> remote arrive round trip"};
  for (int mode = 0; mode < 12; ++mode) {
    const int iters = mode >= 10 ? 1000 : 2000;
    for (int grid : {2, 148}) {
      rate2<<<grid, 128, smem>>>(mode, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("%s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double per = mx / iters;
      double flops;  // per SM (each CTA's 128 rows)
      if (mode <= 2)
        flops = 8.0 * 2 * 128 * (mode == 0 ? 64 : mode == 1 ? 128 : 256) * 16;
      else if (mode == 3)
        flops = 8.0 * 2 * 128 * 128 * 16;
      else if (mode == 4 || mode >= 6)
        flops = 2.0 * (8 * 2.0 * 128 * 64 * 16 + 4 * 2.0 * 128 * 128 * 16);
      else
        flops = 2.0 * (8 * 2.0 * 128 * 128 * 16 + 8 * 2.0 * 128 * 128 * 16);
      if (mode >= 10)
        printf("%-44s grid %3d: %8.1f cycles per round trip\n", names[mode], grid, per);
      else
        printf("%-44s grid %3d: %8.1f cycles per group, %6.0f flop/cycle/SM (%.0f%% of 8192)\n", names[mode], grid,
               per, flops / per, 100.0 * flops / per / 8192);
    }
  }
  return 0;
}
