// tcgen05.mma.kind::i8 throughput probe (M=128, cta_group::1, operands resident in smem):
// one CTA per SM issues R MMAs of 128 x N x 32 into TMEM; reports u8 MAC/s per N.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
template <int N, bool ATMEM, bool MIX = false>
__global__ void bench(int reps, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[4];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * 4096 + 4 * N * 32; i += blockDim.x) smem[i] = (uint8_t)i;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | ((ATMEM ? 0u : 1u) << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = desc(smem_u32(smem), 1024, 128), bd = desc(smem_u32(smem + 4096), (N / 8) * 128, 128);
    auto wait = [&](int r) {  // commit r complete
      asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(smem_u32(&bars[r % 4])), "r"((uint32_t)((r / 4) & 1)));
    };
    for (int r = 0; r < reps; ++r) {
      if (r >= 4) wait(r - 4);  // each barrier phase is waited before its slot is committed again
      for (int i = 0; i < 16; ++i) {
        if constexpr (ATMEM) {
          const uint32_t d = tmem + (uint32_t)((i % (448 / N)) * N);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(tmem + 480u), "l"(bd), "r"(idesc), "r"(1));
        } else if constexpr (MIX) {  // the GEMM's pattern: A plane b, B plane a, shift group a + b
          const int a = i >> 2, b = i & 3;
          const uint64_t ad2 = desc(smem_u32(smem) + b * 4096, 1024, 128);
          const uint64_t bd2 = desc(smem_u32(smem + 4 * 4096) + a * N * 32, (N / 8) * 128, 128);
          const uint32_t d = tmem + (uint32_t)((a + b) * N);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad2), "l"(bd2), "r"(idesc), "r"(1));
        } else {
          const uint32_t d = tmem + (uint32_t)((i % (512 / N)) * N);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[r % 4])));
    }
    for (int r = reps - 4 < 0 ? 0 : reps - 4; r < reps; ++r) wait(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  if (tid == 0 && reps < 0) sink[0] = 1;
}

template <int N, bool ATMEM = false, bool MIX = false>
void run(int sms) {
  const int reps = 2000;
  cudaFuncSetAttribute(bench<N, ATMEM, MIX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  bench<N, ATMEM, MIX><<<sms, 128, 64 * 1024>>>(10, nullptr);
  cudaEventRecord(a);
  bench<N, ATMEM, MIX><<<sms, 128, 64 * 1024>>>(reps, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double macs = (double)sms * reps * 16 * 128.0 * N * 32;
  printf("%s N=%3d: %.3f ms  %.1f T u8-MAC/s  (%.2f POPS)  err=%s\n", ATMEM ? "A:tmem" : MIX ? "mix4x4" : "A:smem", N, ms, macs / ms / 1e9, 2 * macs / ms / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16>(sms);
  run<32>(sms);
  run<64>(sms);
  run<128>(sms);
  run<256>(sms);
  run<16, true>(sms);
  run<32, true>(sms);
  run<64, true>(sms);
  run<16, false, true>(sms);
  run<32, false, true>(sms);
  run<64, false, true>(sms);
  return 0;
}
