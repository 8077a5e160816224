// Integer pipe throughput microbenchmark (sm_100a): ops per clock per SM for
// the instruction classes the codec kernels use.  8 independent chains per
// thread, 32 warps per SM; reported as warp-instructions / cycle / SM.
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed, int iters, long long* cyc) {
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = seed * (threadIdx.x + i + 1);
  const uint32_t c = seed | 1;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(c), "r"(it));
      if constexpr (OP == 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(c), "r"(it));
      if constexpr (OP == 2) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c));
      if constexpr (OP == 3) asm volatile("shf.r.wrap.b32 %0, %0, %0, %1;" : "+r"(r[i]) : "r"(it));
      if constexpr (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x1230;" : "+r"(r[i]) : "r"(c));
      if constexpr (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(c));
      if constexpr (OP == 6) asm volatile("shl.b32 %0, %0, 3;" : "+r"(r[i]));
      if constexpr (OP == 7) asm volatile("shr.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(it));
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* out, long long* cyc, int sms) {
  const int iters = 4096, threads = 1024;
  k<OP><<<sms, threads>>>(out, 3, iters, cyc);
  cudaDeviceSynchronize();
  k<OP><<<sms, threads>>>(out, 3, iters, cyc);
  long long h[1];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double warp_inst = double(iters) * 8 * (threads / 32);
  printf("%-10s %.3f warp-inst/clk/SM\n", name, warp_inst / double(h[0]));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 8);
  run<0>("LOP3", out, cyc, sms);
  run<1>("IMAD", out, cyc, sms);
  run<2>("IMAD.HI", out, cyc, sms);
  run<3>("SHF.var", out, cyc, sms);
  run<4>("PRMT", out, cyc, sms);
  run<5>("IADD", out, cyc, sms);
  run<6>("SHL.imm", out, cyc, sms);
  run<7>("SHR.var", out, cyc, sms);
  return 0;
}
