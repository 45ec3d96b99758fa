// Does a CTA pair (tcgen05.mma.cta_group::2, M = 256, each CTA holding its
// own 128 rows of A and half of B's N columns) cut the conv's per-tile MMA
// cost? Issues the conv's per-tile pattern -- 18 x (N = 64 MMA1, N = 32
// MMA2), A stepping like the conv's shifted taps -- REPS times from one
// thread (the leader's for the pair) and reports cycles per (MMA1, MMA2)
// pair, i.e. per K step, per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2411_16680_b200/csrc profiles/probes/mma2_probe.cu -o /tmp/mma2_probe
#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace lvsg::tc;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}

constexpr int SBO_A = 160, LBO_A = 180 * 16 + 16;

// cta_group::1 reference: one CTA per SM, M = 128
__global__ void __launch_bounds__(128, 1) probe1(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sa = smem_u32(smem), sb = sa + 64 * 1024;
  const uint64_t ah = smem_desc(sa, LBO_A, SBO_A), al = smem_desc(sa + 4 * LBO_A, LBO_A, SBO_A);
  const uint64_t b0 = smem_desc(sb, 64 * 16, 128);
  constexpr uint32_t id64 = idesc_f16(128, 64), id32 = idesc_f16(128, 32);
  if (threadIdx.x < 32) {
    const unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const uint64_t ao = uint64_t((2 * s * LBO_A + ((tap / 3) * 10 + tap % 3) * 16) >> 4);
            const uint64_t bo = uint64_t(((tap * 4 + 2 * s) * 64 * 16) >> 4);
            mma_f16(tmem, ah + ao, b0 + bo, id64, 1u);
            mma_f16(tmem + 32, al + ao, b0 + bo, id32, 1u);
          }
      commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

// cta_group::2: CTA pair, M = 256; B rows split by N between the pair (each
// CTA's descriptor addresses its own half at the same offset)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(256u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sa = smem_u32(smem), sb = sa + 64 * 1024;
  const uint64_t ah = smem_desc(sa, LBO_A, SBO_A), al = smem_desc(sa + 4 * LBO_A, LBO_A, SBO_A);
  // per CTA: 32 rows for MMA1 (N = 64 over the pair), 16 for MMA2 (N = 32)
  const uint64_t b0 = smem_desc(sb, 32 * 16, 128);
  constexpr uint32_t id64 = idesc_f16(256, 64), id32 = idesc_f16(256, 32);
  unsigned long long t0 = 0;
  if (threadIdx.x < 32) {
    t0 = clock64();
    if (rank == 0 && elect_one()) {
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const uint64_t ao = uint64_t((2 * s * LBO_A + ((tap / 3) * 10 + tap % 3) * 16) >> 4);
            const uint64_t bo = uint64_t(((tap * 4 + 2 * s) * 32 * 16) >> 4);
            mma2_f16(tmem, ah + ao, b0 + bo, id64, 1u);
            mma2_f16(tmem + 32, al + ao, b0 + bo, id32, 1u);
          }
      commit2_mc(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  fence_before();
  cluster_sync();
  fence_after();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
}

template <typename K>
void run(const char* name, K kern, int grid, unsigned long long* d, int reps) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  kern<<<grid, 128, 160 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double s = 0;
  int n = 0;
  for (int i = 0; i < grid; ++i)
    if (h[i]) s += double(h[i]), ++n;
  std::printf("{\"probe\": \"%s\", \"cycles_per_k_step\": %.1f, \"ctas\": %d, \"err\": \"%s\"}\n", name,
              n ? s / n / (18.0 * reps) : 0.0, n, cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  cudaMemset(d, 0, sms * sizeof(unsigned long long));
  run("cta_group::1 M=128 (N=64 + N=32)", probe1, sms, d, 200);
  cudaMemset(d, 0, sms * sizeof(unsigned long long));
  run("cta_group::2 M=256 (N=64 + N=32), per pair", probe2, sms, d, 200);
  return 0;
}
