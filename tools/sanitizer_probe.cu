// sanitizer_probe.cu — minimal kernels that reproduce the synchronization patterns of
// span_attn_tc.cu, to tell compute-sanitizer findings about the tool from findings about the
// kernel (profiling aid, not product).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/sanitizer_probe tools/sanitizer_probe.cu -lcuda
//   compute-sanitizer --tool racecheck tools/sanitizer_probe <mode>
//   compute-sanitizer --tool synccheck tools/sanitizer_probe <mode>
//
// mode 0  warp 1 writes buf, arrives E; warp 2 waits E, writes buf        (plain mbarrier order)
// mode 1  warp 1 writes buf, arrives E; warp 0 waits E and issues a bulk copy into buf2 that
//         completes F; warp 2 waits F, writes buf                          (order through the TMA)
// mode 2  as 1, the bulk copy writes buf itself (the Q-slot pattern: epilogue staging -> q_empty
//         -> TMA load -> q_load -> rotation)
// mode 3  mode 0 launched as a programmatic dependent of a long kernel (PDL), the waits ~50 us
//         after the barrier init (the attention kernel launched behind K1)
// mode 4  mode 3 without the PDL attribute
// mode 5  as 2, but warp 1 arrives E from lane 0 only, after __syncwarp (E counts 1): the other
//         lanes' writes are ordered by __syncwarp, not by their own arrive
// mode 6  warp 1 writes buf, arrives E (all lanes); warp 0 (one thread) waits E and arrives F via
//         tcgen05.commit (no MMA pending); warp 2 waits F, writes buf      (order through a commit)
// mode 7  thread 0 initialises 64 barriers; each of warps 1..2 arrives on all of them, warp 3
//         (one elected thread, after setmaxnreg.dec) waits on every one  (synccheck: many barriers)
// mode 8  as 2 with a tensor-map TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B, 4 KB box) instead
//         of a plain bulk copy, and E also counting one tcgen05.commit arrival (the Q-slot ring)
// Every mode is race-free by the PTX memory model (mbarrier.arrive has release, try_wait acquire
// semantics; the bulk copy is issued after the acquiring wait and its complete_tx is observed by
// the second wait). Output: "ok <mode> <checksum>".
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void spin_ns(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); while (t - t0 < ns);
}

__global__ void busy(int* out, uint64_t ns) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  spin_ns(ns);
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

__global__ void __launch_bounds__(96, 1) probe(const float* __restrict__ src, float* __restrict__ out, int mode,
                                               const __grid_constant__ CUtensorMap tm) {
  __shared__ alignas(1024) float tbuf[1024];  // mode 8: 32 rows x 128 B
  __shared__ alignas(128) float buf[32];
  __shared__ alignas(128) float buf2[32];
  __shared__ uint64_t E, F;
  __shared__ uint64_t many[64];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    bar_init(&E, mode == 5 ? 1 : 32);
    bar_init(&F, 1);
    for (int i = 0; i < 64; ++i) bar_init(&many[i], 64);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (mode == 8) {
    if (threadIdx.x == 0) {
      bar_init(&E, 32 + 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (warp == 1) {  // staging writes of 32 rows (one float4 per lane per row)
      for (int r = 0; r < 32; ++r) tbuf[r * 32 + (lane & 31)] = src[lane] + r;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(&E);
    } else if (warp == 0) {
      if (lane == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&E))
                     : "memory");
        bar_wait(&E, 0);
        bar_expect(&F, 4096);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su32(tbuf)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&F)), "r"(0), "r"(0)
            : "memory");
      }
      __syncwarp();
    } else {  // rotation-like read-modify-write of every row
      bar_wait(&F, 0);
      for (int r = 0; r < 32; ++r) tbuf[r * 32 + lane] = tbuf[r * 32 + lane] * 2.f;
      out[lane] = tbuf[lane];
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_slot));
    return;
  }
  if (mode == 6 && warp == 0) {  // tcgen05 needs an allocation before a commit
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (mode == 7) {
    if (warp == 1 || warp == 2) {
      for (int i = 0; i < 64; ++i) bar_arrive(&many[i]);
    } else if (warp == 0) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
      if (lane == 0)
        for (int i = 0; i < 64; ++i) bar_wait(&many[i], 0);
      __syncwarp();
      if (lane == 0) out[0] = 1.f;
    }
    return;
  }
  if (mode >= 3 && mode <= 4) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    spin_ns(50000);
  }
  if (warp == 1) {
    buf[lane] = src[lane] * 2.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode == 5) {
      __syncwarp();
      if (lane == 0) bar_arrive(&E);
    } else {
      bar_arrive(&E);
    }
  } else if (warp == 0 && mode == 6) {
    if (lane == 0) {
      bar_wait(&E, 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&F))
                   : "memory");
    }
    __syncwarp();
  } else if (warp == 0 && (mode == 1 || mode == 2 || mode == 5)) {
    if (lane == 0) {
      bar_wait(&E, 0);
      bar_expect(&F, 128);
      float* dst = mode == 1 ? buf2 : buf;  // modes 2, 5: the copy overwrites buf
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                       su32(dst)),
                   "l"(src + 32), "r"(su32(&F))
                   : "memory");
    }
    __syncwarp();
  } else if (warp == 2) {
    if (mode == 1 || mode == 2 || mode == 5 || mode == 6)
      bar_wait(&F, 0);
    else
      bar_wait(&E, 0);
    buf[lane] = buf[lane] + 1.f;
    out[lane] = buf[lane] + (mode == 1 ? buf2[lane] : 0.f);
  }
  if (mode == 6) {
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_slot));
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  float *src, *out;
  int* tmp;
  cudaMalloc(&src, 64 * sizeof(float));
  cudaMalloc(&out, 32 * sizeof(float));
  cudaMalloc(&tmp, 4096 * sizeof(int));
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = static_cast<float>(i);
  cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const bool pdl_modes = mode == 3 || mode == 4;
  if (pdl_modes) busy<<<sms * 4, 128>>>(tmp, 200000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pdl_modes ? sms : 1);
  cfg.blockDim = dim3(96);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = mode == 3 ? 1 : 0;
  // mode 8: 2D map over a 64 x 64 bf16 matrix, box {64, 32}, SWIZZLE_128B
  CUtensorMap tm{};
  void* big = nullptr;
  cudaMalloc(&big, 64 * 64 * 2);
  cudaMemset(big, 0, 64 * 64 * 2);
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    cuuint64_t dims[2] = {64, 64}, strides[1] = {128};
    cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
    reinterpret_cast<Fn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, big, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, probe, static_cast<const float*>(src), out, mode, tm);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  float r[32];
  cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
  double cs = 0;
  for (float v : r) cs += v;
  printf("%s %d %.0f\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e), mode, cs);
  return e == cudaSuccess ? 0 : 1;
}
