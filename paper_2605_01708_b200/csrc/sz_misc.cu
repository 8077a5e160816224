// sz_misc.cu — K1 histogram, K7 compare, L0 bit primitives, group coverage,
// K8 synthetic generator, and the shared ABI plumbing (parameter validation,
// CUDA error capture).
#include <cstdio>
#include <cstring>

#include "sz_common.cuh"

namespace sz {

// ------------------------------------------------------------------ K1
// build_histogram (calibration.py:79-85).  Privatised shared-memory bins,
// [copy][bin][lane]: lane l increments column l of its copy, so the 32
// atomics of a warp instruction hit 32 distinct words in 32 distinct banks —
// one pass, whatever the (skewed: one bin holds ~28% of KV exponents)
// distribution.  BF16 shares one 256 x 32 copy (32 KiB) per CTA among its
// warps (several CTAs per SM); FP8 keeps a copy per warp (4 KiB / 2 KiB).
// Bins are merged per CTA and added to the (pre-zeroed) global u64 counts.
template <int FMT>
struct HistCfg {
  static constexpr int kBins = 1 << Fmt<FMT>::kExpBits;
  static constexpr int kCols = 32;
  static constexpr int kCopies = FMT == SZ_BF16 ? 1 : kWarps;
  static constexpr int kSmemWords = kCopies * kBins * kCols;
};

template <int FMT>
__device__ __forceinline__ void hist_vec(uint32_t* h, const uint32_t (&x)[8]) {
  constexpr int kCols = HistCfg<FMT>::kCols;
  // h already points at column `lane` of this warp's copy
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    if constexpr (FMT == SZ_BF16) {
      atomicAdd(&h[((x[w] >> 7) & 0xFF) * kCols], 1u);
      atomicAdd(&h[((x[w] >> 23) & 0xFF) * kCols], 1u);
    } else {
      constexpr int sh = FMT == SZ_E5M2 ? 2 : 3;
      constexpr uint32_t mk = FMT == SZ_E5M2 ? 0x1F : 0x0F;
#pragma unroll
      for (int b = 0; b < 4; ++b) atomicAdd(&h[((x[w] >> (8 * b + sh)) & mk) * kCols], 1u);
    }
  }
}

template <int FMT>
__global__ void __launch_bounds__(kThreads) hist_kernel(const uint8_t* __restrict__ words,
                                                        uint64_t n,
                                                        unsigned long long* __restrict__ counts) {
  using C = HistCfg<FMT>;
  constexpr int EPV = kEpv<FMT>;
  constexpr int WB = Fmt<FMT>::kWordBytes;
#ifndef SZ_K1_UNROLL
#define SZ_K1_UNROLL 8
#endif
  constexpr int UNROLL = SZ_K1_UNROLL;
  extern __shared__ uint32_t hsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < C::kSmemWords; i += kThreads) hsm[i] = 0;
  __syncthreads();
  uint32_t* h = hsm + (warp % C::kCopies) * C::kBins * C::kCols + lane;
  const uint64_t nvec = n / EPV;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  uint64_t v = static_cast<uint64_t>(blockIdx.x) * kThreads + tid;
  for (; v + (UNROLL - 1) * stride < nvec; v += UNROLL * stride) {
    uint32_t x[UNROLL][8];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) ld_stream256(words + (v + u * stride) * 32, x[u]);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) hist_vec<FMT>(h, x[u]);
  }
  for (; v < nvec; v += stride) {
    uint32_t x[8];
    ld_stream256(words + v * 32, x);
    hist_vec<FMT>(h, x);
  }
  if (blockIdx.x == 0) {  // ragged tail (< EPV elements)
    for (uint64_t i = nvec * EPV + tid; i < n; i += kThreads) {
      uint32_t w = WB == 2 ? reinterpret_cast<const uint16_t*>(words)[i] : words[i];
      uint32_t e = FMT == SZ_BF16 ? (w >> 7) & 0xFF : (FMT == SZ_E5M2 ? (w >> 2) & 0x1F : (w >> 3) & 0xF);
      atomicAdd(&h[e * C::kCols], 1u);
    }
  }
  __syncthreads();
  for (int b = tid; b < C::kBins; b += kThreads) {
    unsigned long long sum = 0;
    for (int w = 0; w < C::kCopies; ++w)
      for (int c = 0; c < C::kCols; ++c)  // (rotated start: no bank conflicts)
        sum += hsm[(w * C::kBins + b) * C::kCols + ((c + b) & (C::kCols - 1))];
    if (sum) atomicAdd(&counts[b], sum);
  }
}

// ------------------------------------------------------------------ K7
// compare_streams (codec.py:572-581): mismatching words + first mismatch.
template <int WB>
__global__ void __launch_bounds__(kThreads) compare_kernel(const uint8_t* __restrict__ a,
                                                           const uint8_t* __restrict__ b,
                                                           uint64_t n, uint64_t* result) {
  constexpr int EPV = 32 / WB;
  __shared__ unsigned long long s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const uint64_t nvec = n / EPV;
  unsigned long long cnt = 0;
  uint64_t first = ~0ull;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; v < nvec;
       v += static_cast<uint64_t>(gridDim.x) * kThreads) {
    uint32_t x[8], y[8];
    ld_stream256(a + v * 32, x);
    ld_stream256(b + v * 32, y);
    uint32_t vm = 0;  // bit per word-element
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t d = x[w] ^ y[w];
      if constexpr (WB == 2) {
        vm |= (((d & 0xFFFFu) != 0) | (((d >> 16) != 0) << 1)) << (2 * w);
      } else {
        uint32_t t = d | (d >> 4);
        t |= t >> 2;
        t |= t >> 1;
        t &= 0x01010101u;
        vm |= ((t * 0x01020408u) >> 24) << (4 * w);
      }
    }
    if (vm) {
      cnt += __popc(vm);
      first = min(first, v * EPV + (__ffs(vm) - 1));
    }
  }
  if (blockIdx.x == 0) {
    for (uint64_t i = nvec * EPV + threadIdx.x; i < n; i += kThreads) {
      bool diff = WB == 2 ? reinterpret_cast<const uint16_t*>(a)[i] != reinterpret_cast<const uint16_t*>(b)[i]
                          : a[i] != b[i];
      if (diff) {
        ++cnt;
        first = min(first, i);
      }
    }
  }
  if (cnt) atomicAdd(&s_cnt, cnt);
  if (first != ~0ull) record_first(&result[1], first);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) atomicAdd(reinterpret_cast<unsigned long long*>(&result[0]), s_cnt);
}

// ------------------------------------------------------- L0 primitives
__global__ void split_kernel(const uint8_t* __restrict__ words, uint64_t n, uint32_t fmt,
                             uint8_t* __restrict__ exp, uint8_t* __restrict__ sm) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (fmt == SZ_BF16) {
      const uint32_t w = reinterpret_cast<const uint16_t*>(words)[i];
      exp[i] = (w >> 7) & 0xFF;
      sm[i] = ((w >> 8) & 0x80) | (w & 0x7F);
    } else if (fmt == SZ_E5M2) {
      const uint32_t w = words[i];
      exp[i] = (w >> 2) & 0x1F;
      sm[i] = ((w >> 7) << 2) | (w & 3);
    } else {
      const uint32_t w = words[i];
      exp[i] = (w >> 3) & 0x0F;
      sm[i] = ((w >> 7) << 3) | (w & 7);
    }
  }
}

__global__ void reconstruct_kernel(const uint8_t* __restrict__ exp, const uint8_t* __restrict__ sm,
                                   uint64_t n, uint32_t fmt, uint8_t* __restrict__ words) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = exp[i], a = sm[i];
    if (fmt == SZ_BF16) {
      reinterpret_cast<uint16_t*>(words)[i] =
          static_cast<uint16_t>(((a & 0x80) << 8) | ((e & 0xFF) << 7) | (a & 0x7F));
    } else if (fmt == SZ_E5M2) {
      words[i] = static_cast<uint8_t>((((a >> 2) & 1) << 7) | ((e & 0x1F) << 2) | (a & 3));
    } else {
      words[i] = static_cast<uint8_t>((((a >> 3) & 1) << 7) | ((e & 0x0F) << 3) | (a & 7));
    }
  }
}

// 8 symbols -> `width` bytes per thread (LSB-first stream, formats.py:8-19).
__global__ void pack_bits_kernel(const uint8_t* __restrict__ sym, uint64_t n, int width,
                                 uint8_t* __restrict__ out) {
  const uint64_t groups = (n + 7) / 8, nbytes = (n * width + 7) / 8;
  const uint32_t mask = (1u << width) - 1;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < groups;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t acc = 0;
    for (int j = 0; j < 8; ++j) {
      const uint64_t i = g * 8 + j;
      if (i < n) acc |= static_cast<uint64_t>(sym[i] & mask) << (j * width);
    }
    for (int b = 0; b < width; ++b)
      if (g * width + b < nbytes) out[g * width + b] = static_cast<uint8_t>(acc >> (8 * b));
  }
}

__global__ void unpack_bits_kernel(const uint8_t* __restrict__ packed, uint64_t n, int width,
                                   uint8_t* __restrict__ sym, uint32_t* pad_nonzero) {
  const uint64_t groups = (n + 7) / 8, nbytes = (n * width + 7) / 8;
  const uint32_t mask = (1u << width) - 1;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < groups;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t acc = 0;
    for (int b = 0; b < width; ++b)
      if (g * width + b < nbytes) acc |= static_cast<uint64_t>(packed[g * width + b]) << (8 * b);
    for (int j = 0; j < 8; ++j) {
      const uint64_t i = g * 8 + j;
      if (i < n) sym[i] = static_cast<uint8_t>((acc >> (j * width)) & mask);
    }
    if (g == groups - 1) {
      const uint64_t used = n * width - g * 8 * width;  // bits of this group in use
      if (used < 64 && (acc >> used)) atomicOr(pad_nonzero, 1u);
    }
  }
}

__global__ void max_u8_kernel(const uint8_t* __restrict__ in, uint64_t n, uint32_t* out) {
  uint32_t mx = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    mx = max(mx, static_cast<uint32_t>(in[i]));
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// coverage_by_group (calibration.py:191-212): member count per group.
__global__ void group_members_kernel(const uint8_t* __restrict__ words, uint64_t n,
                                     const __grid_constant__ sz_params p, uint64_t group,
                                     unsigned long long* hits) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t e;
    if (p.fmt == SZ_BF16) e = (reinterpret_cast<const uint16_t*>(words)[i] >> 7) & 0xFF;
    else if (p.fmt == SZ_E5M2) e = (words[i] >> 2) & 0x1F;
    else e = (words[i] >> 3) & 0xF;
    const bool member = !(p.enc_lut[e] & 0x10);
    // aggregate equal groups across the warp
    const uint64_t gi = i / group;
    const uint32_t active = __activemask();
    const uint32_t same = __match_any_sync(active, gi);
    const uint32_t votes = __ballot_sync(active, member) & same;
    if ((__ffs(same) - 1) == static_cast<int>(threadIdx.x & 31) && votes)
      atomicAdd(&hits[gi], static_cast<unsigned long long>(__popc(votes)));
  }
}

// ------------------------------------------------------------------ K8
// Counter-based synthetic KV words: exponent drawn from a CDF table (the
// distribution of datagen.generate's sampled mode, datagen.py:116-122),
// sign|mantissa uniform (datagen.py:124).  Deterministic in (seed, index).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct SynthTable {
  uint8_t exps[64];
  uint32_t cdf[64];
  uint32_t count;
};

template <int WB>
__global__ void __launch_bounds__(kThreads) synth_kernel(uint8_t* __restrict__ out, uint64_t n,
                                                         uint32_t fmt, uint64_t seed,
                                                         const __grid_constant__ SynthTable t) {
  __shared__ uint32_t cdf[64];
  __shared__ uint8_t ex[64];
  if (threadIdx.x < 64) {
    cdf[threadIdx.x] = t.cdf[threadIdx.x];
    ex[threadIdx.x] = t.exps[threadIdx.x];
  }
  __syncthreads();
  constexpr int EPV = 32 / WB;
  const uint64_t nvec = (n + EPV - 1) / EPV;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; v < nvec;
       v += static_cast<uint64_t>(gridDim.x) * kThreads) {
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < EPV; ++j) {
      const uint64_t i = v * EPV + j;
      const uint64_t r = mix64(seed * 0x9E3779B97F4A7C15ull + i);
      const uint32_t u = static_cast<uint32_t>(r);
      uint32_t k = 0;
      while (k + 1 < t.count && u > cdf[k]) ++k;
      const uint32_t e = ex[k], a = static_cast<uint32_t>(r >> 40) & 0xFF;
      uint32_t word;
      if (fmt == SZ_BF16) word = ((a & 0x80) << 8) | (e << 7) | (a & 0x7F);
      else if (fmt == SZ_E5M2) word = (((a >> 2) & 1) << 7) | ((e & 0x1F) << 2) | (a & 3);
      else word = (((a >> 3) & 1) << 7) | ((e & 0xF) << 3) | (a & 7);
      w[(j * WB) >> 2] |= word << (8 * ((j * WB) & 3));
    }
    if ((v + 1) * EPV <= n) {
      st256(out + v * 32, w);
    } else {
      st_bytes_clipped<32>(out, v * 32, w, n * WB);
    }
  }
}

}  // namespace sz

// ============================================================ C ABI
using namespace sz;

static thread_local char g_last_error[256] = "";

namespace {
int grid_for(uint64_t work, int per_block) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 148ull * 16) g = 148ull * 16;
  return static_cast<int>(g);
}
int check(cudaError_t e);
}  // namespace

extern "C" {

int sz_record_cuda(cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return SZ_ECUDA;
}

int sz_check_params(const sz_params* p, int decode_side) {
  (void)decode_side;
  if (!p) return SZ_ECONFIG;
  if (p->fmt > SZ_E4M3 || (p->code_bits != 3 && p->code_bits != 4)) return SZ_ECONFIG;
  if (p->chunk_size < 1) return SZ_ECONFIG;
  const bool chunked = !p->sentinel && !p->abs32;
  if (chunked && p->chunk_size > 65536) return SZ_ECONFIG;
  if (p->sentinel && p->abs32) return SZ_ECONFIG;
  const uint32_t cap = (1u << p->code_bits) - (p->sentinel ? 1u : 0u);
  if (p->n_entries > cap) return SZ_ECONFIG;
  return SZ_OK;
}

int sz_abi_version(void) { return SZ_ABI_VERSION; }
const char* sz_last_cuda_error(void) { return g_last_error; }

int sz_split_fields(const void* d_words, uint64_t n, uint32_t fmt, uint8_t* d_exp, uint8_t* d_sm,
                    void* stream) {
  if (fmt > SZ_E4M3) return SZ_ECONFIG;
  if (!n) return SZ_OK;
  split_kernel<<<grid_for(n, 1024), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(d_words), n, fmt, d_exp, d_sm);
  return check(cudaGetLastError());
}

int sz_reconstruct(const uint8_t* d_exp, const uint8_t* d_sm, uint64_t n, uint32_t fmt,
                   void* d_words, void* stream) {
  if (fmt > SZ_E4M3) return SZ_ECONFIG;
  if (!n) return SZ_OK;
  reconstruct_kernel<<<grid_for(n, 1024), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      d_exp, d_sm, n, fmt, static_cast<uint8_t*>(d_words));
  return check(cudaGetLastError());
}

int sz_pack_bits(const uint8_t* d_symbols, uint64_t n, uint32_t width, uint8_t* d_out,
                 void* stream) {
  if (width < 1 || width > 8) return SZ_ECONFIG;
  if (!n) return SZ_OK;
  pack_bits_kernel<<<grid_for((n + 7) / 8, kThreads), kThreads, 0,
                     static_cast<cudaStream_t>(stream)>>>(d_symbols, n, width, d_out);
  return check(cudaGetLastError());
}

int sz_unpack_bits(const uint8_t* d_packed, uint64_t n, uint32_t width, uint8_t* d_symbols,
                   uint32_t* d_pad_nonzero, void* stream) {
  if (width < 1 || width > 8) return SZ_ECONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_pad_nonzero, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (!n) return SZ_OK;
  unpack_bits_kernel<<<grid_for((n + 7) / 8, kThreads), kThreads, 0, s>>>(d_packed, n, width,
                                                                          d_symbols, d_pad_nonzero);
  return check(cudaGetLastError());
}

int sz_max_u8(const uint8_t* d_in, uint64_t n, uint32_t* d_max, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_max, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (!n) return SZ_OK;
  max_u8_kernel<<<grid_for(n, 4096), kThreads, 0, s>>>(d_in, n, d_max);
  return check(cudaGetLastError());
}

size_t sz_histogram_workspace_bytes(uint64_t n, uint32_t fmt) {
  (void)n;
  (void)fmt;
  return 0;
}

int sz_histogram(const void* d_words, uint64_t n, uint32_t fmt, uint64_t* d_counts, void* d_ws,
                 size_t ws_bytes, void* stream) {
  (void)d_ws;
  (void)ws_bytes;
  if (fmt > SZ_E4M3 || !d_counts) return SZ_ECONFIG;
  if (reinterpret_cast<uintptr_t>(d_words) & 31) return SZ_EALIGN;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int bins = fmt == SZ_BF16 ? 256 : (fmt == SZ_E5M2 ? 32 : 16);
  cudaError_t e = cudaMemsetAsync(d_counts, 0, bins * sizeof(uint64_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (!n) return SZ_OK;
  auto launch = [&](auto kern, int smem_words, uint64_t epv) {
    const size_t smem = static_cast<size_t>(smem_words) * 4;
    const KernelSetup ks = kernel_setup(reinterpret_cast<const void*>(kern),
                                        static_cast<int>(smem), kThreads);
    uint64_t want = (n / epv + kThreads - 1) / kThreads;
    uint64_t cap = static_cast<uint64_t>(ks.sms) * (ks.per_sm > 0 ? ks.per_sm : 1);
    unsigned grid = static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
    kern<<<grid, kThreads, smem, s>>>(static_cast<const uint8_t*>(d_words), n,
                                      reinterpret_cast<unsigned long long*>(d_counts));
  };
  switch (fmt) {
    case SZ_BF16: launch(hist_kernel<SZ_BF16>, HistCfg<SZ_BF16>::kSmemWords, 16); break;
    case SZ_E5M2: launch(hist_kernel<SZ_E5M2>, HistCfg<SZ_E5M2>::kSmemWords, 32); break;
    default: launch(hist_kernel<SZ_E4M3>, HistCfg<SZ_E4M3>::kSmemWords, 32); break;
  }
  return check(cudaGetLastError());
}

int sz_compare(const void* d_a, const void* d_b, uint64_t n, uint32_t word_bytes,
               uint64_t* d_result, void* stream) {
  if (word_bytes != 1 && word_bytes != 2) return SZ_ECONFIG;
  if ((reinterpret_cast<uintptr_t>(d_a) & 31) || (reinterpret_cast<uintptr_t>(d_b) & 31))
    return SZ_EALIGN;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_result, 0, 2 * sizeof(uint64_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (!n) return SZ_OK;
  const int grid = grid_for(n * word_bytes, 32 * kThreads * 4);
  if (word_bytes == 2)
    compare_kernel<2><<<grid, kThreads, 0, s>>>(static_cast<const uint8_t*>(d_a),
                                                static_cast<const uint8_t*>(d_b), n, d_result);
  else
    compare_kernel<1><<<grid, kThreads, 0, s>>>(static_cast<const uint8_t*>(d_a),
                                                static_cast<const uint8_t*>(d_b), n, d_result);
  return check(cudaGetLastError());
}

int sz_group_members(const void* d_words, uint64_t n, const sz_params* p, uint64_t group,
                     uint64_t* d_hits, void* stream) {
  if (sz_check_params(p, 0) || group < 1) return SZ_ECONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t ngroups = (n + group - 1) / group;
  cudaError_t e = cudaMemsetAsync(d_hits, 0, ngroups * sizeof(uint64_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (!n) return SZ_OK;
  group_members_kernel<<<grid_for(n, 4096), kThreads, 0, s>>>(
      static_cast<const uint8_t*>(d_words), n, *p, group,
      reinterpret_cast<unsigned long long*>(d_hits));
  return check(cudaGetLastError());
}

int sz_synth_words(void* d_words, uint64_t n, uint32_t fmt, uint64_t seed, const uint8_t* exps,
                   const uint32_t* cdf_q32, uint32_t n_exps, void* stream) {
  if (fmt > SZ_E4M3 || n_exps < 1 || n_exps > 64) return SZ_ECONFIG;
  if (reinterpret_cast<uintptr_t>(d_words) & 31) return SZ_EALIGN;
  if (!n) return SZ_OK;
  SynthTable t{};
  std::memcpy(t.exps, exps, n_exps);
  std::memcpy(t.cdf, cdf_q32, n_exps * sizeof(uint32_t));
  t.count = n_exps;
  const uint64_t epv = fmt == SZ_BF16 ? 16 : 32;
  const int grid = grid_for((n + epv - 1) / epv, kThreads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fmt == SZ_BF16)
    synth_kernel<2><<<grid, kThreads, 0, s>>>(static_cast<uint8_t*>(d_words), n, fmt, seed, t);
  else
    synth_kernel<1><<<grid, kThreads, 0, s>>>(static_cast<uint8_t*>(d_words), n, fmt, seed, t);
  return check(cudaGetLastError());
}

}  // extern "C"

namespace {
int check(cudaError_t e) { return e == cudaSuccess ? SZ_OK : sz_record_cuda(e); }
}  // namespace
