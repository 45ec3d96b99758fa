// Cost of one tcgen05.mma.kind::f16 (A and B from shared memory, fp32
// accumulate) by shape: one CTA per SM issues REPS x 36 MMAs (the conv's
// per-tile count) back to back from one thread, A start address stepping by
// 16 bytes like the conv's shifted taps; cycles from first issue to the
// commit's mbarrier completion. Prints cycles per MMA for each (M, N).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//        -I paper_2411_16680_b200/csrc profiles/probes/mma_probe.cu -o /tmp/mma_probe
#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace lvsg::tc;

template <int M, int N, int SBO_A, bool VARY_B>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sa = smem_u32(smem), sb = sa + 16 * 1024;
  // K-major interleave: 8-row x 16-byte core matrices, 128 B apart along
  // M/N (SBO), the two K chunks M*16 (resp. N*16) bytes apart (LBO)
  // A core matrices SBO_A bytes apart along M (128: dense; 160: the conv's
  // halo-row pitch, 10 pixels x 16 B; 256: a padded pitch), LBO after them
  const uint64_t a0 = smem_desc(sa, (M / 8) * SBO_A, SBO_A);
  const uint64_t b0 = smem_desc(sb, N * 16, 128);
  constexpr uint32_t id = idesc_f16(M, N);
  if (threadIdx.x < 32) {
    const unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int i = 0; i < 36; ++i)
          mma_f16(tmem, a0 + uint64_t(i % 9), VARY_B ? b0 + uint64_t((i * N * 32) >> 4) : b0, id, 1u);
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
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int M, int N, int SBO_A = 128, bool VARY_B = false>
void run(int sms, unsigned long long* d, int reps) {
  cudaFuncSetAttribute(probe<M, N, SBO_A, VARY_B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       160 * 1024);
  probe<M, N, SBO_A, VARY_B><<<sms, 128, 160 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double s = 0;
  for (auto v : h) s += double(v);
  const double per = s / sms / (36.0 * reps);
  const double macs = double(M) * N * 16;
  std::printf("{\"M\": %d, \"N\": %d, \"sbo_a\": %d, \"vary_b\": %d, \"cycles_per_mma\": %.1f, \"macs_per_cycle\": %.0f, \"err\": \"%s\"}\n",
              M, N, SBO_A, int(VARY_B), per, macs / per, cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int reps = 200;
  run<128, 32>(sms, d, reps);
  run<128, 64>(sms, d, reps);
  run<128, 128>(sms, d, reps);
  run<128, 256>(sms, d, reps);
  run<64, 64>(sms, d, reps);
  run<64, 128>(sms, d, reps);
  run<64, 256>(sms, d, reps);
  run<128, 32, 160>(sms, d, reps);
  run<128, 64, 160>(sms, d, reps);
  run<128, 32, 256>(sms, d, reps);
  run<128, 64, 256>(sms, d, reps);
  run<128, 32, 160, true>(sms, d, reps);
  run<128, 64, 160, true>(sms, d, reps);
  run<128, 128, 160, true>(sms, d, reps);
  return 0;
}
