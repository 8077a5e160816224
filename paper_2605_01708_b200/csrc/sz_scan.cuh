// sz_scan.cuh — exclusive u64 scan of u32 counts (K3 of the decoder: chunk
// escape counts -> chunk ordinal offsets, codec.py:491-536's prefix; the
// encoder's K2b uses it for the per-tile escape prefix).
//
// Single pass, decoupled look-back (lookback_warp) across CTAs of 4096
// counts.  Warp-contiguous layout: row r of warp w is 128 consecutive counts,
// lane l holding counts 4l..4l+3 of it, so every load (uint4) and every store
// (2 x uint4 of u64 prefixes) of a warp covers one contiguous span — the
// earlier thread-contiguous layout (64 counts per thread) spread each warp
// access over 32 lines and ran at ~0.3 TB/s.
#pragma once
#include "sz_common.cuh"

namespace sz {
namespace {

struct OffsetsArgs {
  const uint64_t* m_ptr;
  const uint32_t* counts;
  uint64_t n_counts;
  uint64_t m;
  uint64_t* offsets;      // n_counts + 1 entries (offsets[n_counts] = total)
  uint64_t* states;
  unsigned long long* tile_counter;
  uint64_t num_tiles;
  sz_decode_status* status;  // null: plain scan (no count-total check)
  int32_t sentinel;          // counts are per-tile sentinel marks (codec.py:459-467)
  // reduce-then-scan (many CTAs): per-CTA sums from offsets_sums_kernel; the
  // exclusive prefix of CTA t is then the sum of sums[0..t) — no look-back
  const uint64_t* sums;
};

constexpr int kScanRows = 8;                          // rows of 128 counts per warp
constexpr int kScanPerWarp = kScanRows * 128;
constexpr int kScanPerCta = kScanPerWarp * kWarps;    // 8192 counts per CTA

inline uint64_t offsets_tiles(uint64_t n_counts) {
  return (n_counts + kScanPerCta - 1) / kScanPerCta;
}

// Loads one CTA's counts in the warp-contiguous layout.
__device__ __forceinline__ void scan_load(const OffsetsArgs& a, uint64_t wbase,
                                          uint32_t (&c)[kScanRows][4]) {
  const int lane = threadIdx.x & 31;
  const uint64_t n = a.n_counts;
  const bool vin = !(reinterpret_cast<uintptr_t>(a.counts) & 15);
#pragma unroll
  for (int r = 0; r < kScanRows; ++r) {
    const uint64_t idx = wbase + r * 128 + lane * 4;
    if (vin && idx + 4 <= n) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(a.counts + idx));
      c[r][0] = q.x; c[r][1] = q.y; c[r][2] = q.z; c[r][3] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) c[r][k] = idx + k < n ? a.counts[idx + k] : 0u;
    }
  }
}

// Reduce pass of the reduce-then-scan: the u64 sum of each CTA's counts.
__global__ void __launch_bounds__(kThreads) offsets_sums_kernel(const OffsetsArgs a,
                                                                uint64_t* sums) {
  __shared__ uint64_t wsum[kWarps];
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t wbase = blockIdx.x * static_cast<uint64_t>(kScanPerCta) +
                         static_cast<uint64_t>(warp) * kScanPerWarp;
  uint32_t c[kScanRows][4];
  scan_load(a, wbase, c);
  uint64_t t = 0;
#pragma unroll
  for (int r = 0; r < kScanRows; ++r)
    t += static_cast<uint64_t>(c[r][0]) + c[r][1] + c[r][2] + c[r][3];
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
  if (lane == 0) wsum[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += wsum[w];
    sums[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) offsets_kernel(const OffsetsArgs a) {
  __shared__ uint64_t warp_tot[kWarps];
  __shared__ unsigned long long s_tile;
  __shared__ uint64_t s_excl, s_total;
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!a.sums) {
    if (tid == 0) s_tile = atomicAdd(a.tile_counter, 1ull);
    __syncthreads();
  }
  const uint64_t tile = a.sums ? blockIdx.x : s_tile;
  const uint64_t n = a.n_counts;
  const uint64_t wbase = tile * kScanPerCta + static_cast<uint64_t>(warp) * kScanPerWarp;
  const bool vout = !(reinterpret_cast<uintptr_t>(a.offsets) & 15);
  uint32_t c[kScanRows][4];
  scan_load(a, wbase, c);
  // reduce-then-scan: this CTA's prefix = the sums of the CTAs before it
  uint64_t pre = 0;
  if (a.sums) {
    for (uint64_t i = tid; i < tile; i += kThreads) pre += a.sums[i];
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, d);
  }
  // per row: lane sums and their warp scan (u64: corrupt counts may be huge)
  uint64_t sum[kScanRows], incl[kScanRows], rowtot[kScanRows];
  uint64_t wtot = 0;
#pragma unroll
  for (int r = 0; r < kScanRows; ++r) {
    sum[r] = static_cast<uint64_t>(c[r][0]) + c[r][1] + c[r][2] + c[r][3];
    uint64_t x = sum[r];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t o = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += o;
    }
    incl[r] = x;
    rowtot[r] = __shfl_sync(0xffffffffu, x, 31);
    wtot += rowtot[r];
  }
  __shared__ uint64_t pre_w[kWarps];
  if (lane == 0) {
    warp_tot[warp] = wtot;
    pre_w[warp] = pre;
  }
  __syncthreads();
  if (warp == 0) {
    const uint64_t w = lane < kWarps ? warp_tot[lane] : 0;
    uint64_t xw = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t o = __shfl_up_sync(0xffffffffu, xw, d);
      if (lane >= d) xw += o;
    }
    const uint64_t total = __shfl_sync(0xffffffffu, xw, 31);
    uint64_t ex;
    if (a.sums) {
      uint64_t pw = lane < kWarps ? pre_w[lane] : 0;
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, d);
      ex = pw;
    } else {
      ex = lookback_warp(a.states, tile, total);
    }
    if (lane < kWarps) warp_tot[lane] = xw - w;
    if (lane == 0) {
      s_excl = ex;
      s_total = ex + total;
    }
  }
  __syncthreads();
  uint64_t run = s_excl + warp_tot[warp];
#pragma unroll
  for (int r = 0; r < kScanRows; ++r) {
    const uint64_t idx = wbase + r * 128 + lane * 4;
    const uint64_t o0 = run + incl[r] - sum[r], o1 = o0 + c[r][0], o2 = o1 + c[r][1],
                   o3 = o2 + c[r][2];
    if (vout && idx + 4 <= n) {
      uint4* dst = reinterpret_cast<uint4*>(a.offsets + idx);
      dst[0] = make_uint4(static_cast<uint32_t>(o0), static_cast<uint32_t>(o0 >> 32),
                          static_cast<uint32_t>(o1), static_cast<uint32_t>(o1 >> 32));
      dst[1] = make_uint4(static_cast<uint32_t>(o2), static_cast<uint32_t>(o2 >> 32),
                          static_cast<uint32_t>(o3), static_cast<uint32_t>(o3 >> 32));
    } else {
      const uint64_t o[4] = {o0, o1, o2, o3};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (idx + k < n) a.offsets[idx + k] = o[k];
    }
    run += rowtot[r];
  }
  if (tile == a.num_tiles - 1 && tid == 0) {
    a.offsets[n] = s_total;
    if (a.status) {
      const uint64_t m = a.m_ptr ? min(*a.m_ptr, a.m) : a.m;
      if (a.sentinel) {
        a.status->marks_total = s_total;
        if (s_total != m) atomicOr(&a.status->flags, 1u << SZ_DEC_SENTINEL_COUNT);
      } else {
        a.status->counts_total = s_total;
        if (s_total != m) atomicOr(&a.status->flags, 1u << SZ_DEC_COUNTS_TOTAL);
      }
    }
  }
}

}  // namespace
}  // namespace sz
