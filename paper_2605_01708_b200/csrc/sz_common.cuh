// sz_common.cuh — device helpers shared by the SplitZip sm_100a kernels.
//
// Everything here is integer/bitwise work; nothing touches tensor cores.  The
// kernels are HBM-bound streams, so the helpers are about moving bytes:
// 256-bit global loads/stores (LDG.E.256 / STG.E.256 on sm_100a), a block-wide
// exclusive scan in (item, thread) order, and a decoupled look-back over a
// per-call tile-state array (flag and value packed into one 64-bit word so a
// single relaxed store publishes both atomically).
#pragma once

#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <cuda_runtime.h>

#include "../../include/splitzip_b200.h"

// Per-role cycle counters for pipeline tuning (build with -DSZ_TIMERS and run
// with SZ_DEBUG_TIMERS=1); compiled out otherwise.
#ifdef SZ_TIMERS
#define SZ_CLOCK() clock64()
#else
#define SZ_CLOCK() 0ll
#endif

namespace sz {

// ---------------------------------------------------------------- launch setup
// Per (kernel, device): raise the dynamic shared-memory limit once and cache
// the occupancy and SM count, so a launch costs no attribute calls (a 64 MiB
// handoff piece encodes in ~18 us of device time; per-call
// cudaFuncSetAttribute + occupancy queries were a visible share of it).
// SM count of the current device, cached per device ordinal.
inline int device_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = sms;
  }
  return cached[dev];
}

struct KernelSetup {
  cudaError_t err;
  int per_sm;  // resident CTAs per SM at (threads, smem)
  int sms;
};
inline KernelSetup kernel_setup(const void* kern, int smem, int threads) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, KernelSetup> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(kern) << 8) ^ static_cast<uint64_t>(dev) ^
                       (static_cast<uint64_t>(smem) << 48) ^ (static_cast<uint64_t>(threads) << 40);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  KernelSetup k{cudaSuccess, 1, 148};
  if (smem > 0)
    k.err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (k.err == cudaSuccess) {
    int per_sm = 0;
    k.err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    k.per_sm = per_sm;
  }
  cudaDeviceGetAttribute(&k.sms, cudaDevAttrMultiProcessorCount, dev);
  if (k.err == cudaSuccess) {
    std::lock_guard<std::mutex> g(mu);
    cache.emplace(key, k);
  }
  return k;
}

constexpr int kThreads = 256;          // CTA size of every streaming kernel
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------- formats
// (word bytes, exponent bits, sign|mantissa bits) — formats.py:49-51.
template <int FMT> struct Fmt;
template <> struct Fmt<SZ_BF16> {
  static constexpr int kWordBytes = 2, kExpBits = 8, kSmBits = 8;
};
template <> struct Fmt<SZ_E5M2> {
  static constexpr int kWordBytes = 1, kExpBits = 5, kSmBits = 3;
};
template <> struct Fmt<SZ_E4M3> {
  static constexpr int kWordBytes = 1, kExpBits = 4, kSmBits = 4;
};
// Elements per 32-byte vector ("slot").
template <int FMT> constexpr int kEpv = 32 / Fmt<FMT>::kWordBytes;

// ---------------------------------------------------------- memory access
__device__ __forceinline__ void ld_stream256(const void* p, uint32_t (&r)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7])
      : "l"(p));
}
__device__ __forceinline__ void st256(void* p, const uint32_t (&r)[8]) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ uint4 ld_stream128(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ld_stream64(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Store `nbytes` (multiple of 2, <= 16) from packed words; the destination is
// aligned to the largest power of two dividing nbytes.
template <int NBYTES>
__device__ __forceinline__ void st_packed(uint8_t* dst, const uint32_t* w) {
  if constexpr (NBYTES == 16) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  } else if constexpr (NBYTES == 12) {
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    d[0] = w[0]; d[1] = w[1]; d[2] = w[2];
  } else if constexpr (NBYTES == 8) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
  } else if constexpr (NBYTES == 6) {
    uint16_t* d = reinterpret_cast<uint16_t*>(dst);
    d[0] = w[0] & 0xFFFF; d[1] = w[0] >> 16; d[2] = w[1] & 0xFFFF;
  } else {
    static_assert(NBYTES == 16, "unsupported store width");
  }
}
// Byte-granular store clipped to [0, limit) — tail slots only.  Fully
// unrolled so `w` stays in registers.
template <int NBYTES>
__device__ __forceinline__ void st_bytes_clipped(uint8_t* base, uint64_t off,
                                                 const uint32_t* w, uint64_t limit) {
#pragma unroll
  for (int b = 0; b < NBYTES; ++b)
    if (off + b < limit) base[off + b] = (w[b >> 2] >> (8 * (b & 3))) & 0xFF;
}
template <int NBYTES>
__device__ __forceinline__ void ld_bytes_clipped(const uint8_t* base, uint64_t off, uint32_t* w,
                                                 uint64_t limit) {
#pragma unroll
  for (int i = 0; i < (NBYTES + 3) / 4; ++i) w[i] = 0;
#pragma unroll
  for (int b = 0; b < NBYTES; ++b)
    if (off + b < limit) w[b >> 2] |= static_cast<uint32_t>(base[off + b]) << (8 * (b & 3));
}
// Select word k of a small register array without dynamic indexing.
template <int N>
__device__ __forceinline__ uint32_t pick(const uint32_t* w, int k) {
  uint32_t v = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) v = (i == k) ? w[i] : v;
  return v;
}

// -------------------------------------------------------- bit shuffling
// (a & mask) | (b & ~mask) as one LOP3 (ptxas does not always fuse the
// two-constant form).
__device__ __forceinline__ uint32_t bitselect(uint32_t a, uint32_t b, uint32_t mask) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(mask));
  return d;
}
// Four bytes, each < 16, to one 16-bit nibble group (element 0 low nibble) —
// the nibble order of formats.py:180-183.
__device__ __forceinline__ uint32_t pack_nib4(uint32_t b4) {
  uint32_t t = b4 | (b4 >> 4);
  return __byte_perm(t, 0, 0x4420);
}
// Inverses.
__device__ __forceinline__ uint32_t unpack_nib4(uint32_t x16) {
  uint32_t t = __byte_perm(x16, 0, 0x4140);
  return (t | (t << 4)) & 0x0F0F0F0Fu;
}
__device__ __forceinline__ uint32_t unpack_tri4(uint32_t x12) {
  uint32_t u = (x12 | (x12 << 10)) & 0x003F003Fu;
  return (u | (u << 5)) & 0x07070707u;
}
// Append G groups of W bits (W = 12 or 16) into a little-endian stream held
// in `out` (ceil(G*W/32) words).
template <int G, int W>
__device__ __forceinline__ void concat_groups(const uint32_t (&grp)[G], uint32_t* out) {
  constexpr int kWords = (G * W + 31) / 32;
#pragma unroll
  for (int i = 0; i < kWords; ++i) out[i] = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int bit = g * W;
    const int wi = bit >> 5, sh = bit & 31;
    out[wi] |= grp[g] << sh;
    if (sh + W > 32) out[wi + 1] |= grp[g] >> (32 - sh);
  }
}
// Extract group g of W bits from a little-endian stream.
template <int W>
__device__ __forceinline__ uint32_t group_bits(const uint32_t* in, int g) {
  const int bit = g * W;
  const int wi = bit >> 5, sh = bit & 31;
  uint32_t v = in[wi] >> sh;
  if (sh + W > 32) v |= in[wi + 1] << (32 - sh);
  return v & ((1u << W) - 1);
}

// ------------------------------------------------ decoupled look-back
// Tile state word: bits 62-63 flag (0 empty, 1 aggregate, 2 inclusive
// prefix), bits 0-61 value.  The array must be zeroed before the launch.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValueMask = (1ull << 62) - 1;

// Wide look-back: ALL lanes of one warp; every lane reads E predecessor
// states per round (32*E per L2 round trip), so the look-back over W
// concurrently-running tiles costs ceil(W / 32E) round trips instead of W/32.
// The caller's own aggregate must already be published (or tile == 0).
// Returns the exclusive prefix of `tile` in every lane; does not publish.
template <int E>
__device__ __forceinline__ uint64_t lookback_wide(const uint64_t* states, uint64_t tile) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t pred = static_cast<int64_t>(tile) - 1;
  while (pred >= 0) {
    uint64_t st[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int64_t idx = pred - (lane * E + j);
      st[j] = idx >= 0 ? ld_relaxed(&states[idx]) : kFlagPrefix;
    }
    int first = 32 * E;  // distance of the nearest inclusive prefix seen by this lane
#pragma unroll
    for (int j = E - 1; j >= 0; --j)
      if ((st[j] >> 62) == 2) first = lane * E + j;
    first = __reduce_min_sync(0xffffffffu, first);
    bool missing = false;
    uint64_t sum = 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int d = lane * E + j;
      if (d <= first) {
        missing |= (st[j] >> 62) == 0;
        sum += st[j] & kValueMask;
      }
    }
    if (__any_sync(0xffffffffu, missing)) {
      __nanosleep(64);
      continue;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
    excl += sum;
    if (first < 32 * E) break;
    pred -= 32 * E;
  }
  return excl;
}

// Called by ALL lanes of one warp.  Publishes `agg` for `tile`, walks back to
// the nearest inclusive prefix, publishes this tile's inclusive prefix and
// returns the exclusive prefix (in every lane).
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* states, uint64_t tile,
                                                  uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&states[0], kFlagPrefix | agg);
    return 0;
  }
  if (lane == 0) st_relaxed(&states[tile], kFlagAgg | agg);
  __syncwarp();
  const uint64_t excl = lookback_wide<8>(states, tile);
  if (lane == 0) st_relaxed(&states[tile], kFlagPrefix | (excl + agg));
  return excl;
}

// ------------------------------------------------ programmatic dependent launch
// The codec's kernels run back to back on one stream (K2a -> scan -> K2b ->
// K2c, then sums -> K3 -> K4).  Launched with programmatic stream
// serialization (launch_pdl), a kernel's CTAs may be scheduled while its
// predecessor's last CTAs still run: each kernel lets its dependents launch
// at once (pdl_trigger) and waits for its predecessor's completion and
// memory (pdl_wait) before its first global access; only the
// shared-memory prologue overlaps.  Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ------------------------------------------------ mbarrier + TMA bulk copy
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Shared loads from explicit 32-bit shared addresses (lets the caller build
// the address with byte permutes / masks instead of base + index adds).
__device__ __forceinline__ uint32_t lds_u8(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t saddr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}
// 1-D bulk copy global -> shared (TMA engine, UBLKCP), completion counted in
// bytes on `bar`.  src/dst 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Atomic "keep the smallest index" into a zero-initialised slot, storing ~idx.
__device__ __forceinline__ void record_first(uint64_t* slot, uint64_t idx) {
  atomicMax(reinterpret_cast<unsigned long long*>(slot),
            static_cast<unsigned long long>(~idx));
}

}  // namespace sz
