// sz_decode.cu — K3 (chunk offsets) + K4 (decode) for sm_100a.
//
// Replaces codec.py:421-536 (decode, _decode_dense, _escape_indices).
//
// K3: exclusive scan of the u32 per-chunk escape counts into u64 ordinal
//     offsets (the `starts = repeat(chunk*c, counts)` of codec.py:520-523 in
//     prefix form), single pass with decoupled look-back; also checks
//     sum(counts) == M (codec.py:513-514).
// K4: one CTA per tile of ITEMS x 256 x EPV elements:
//   - vector loads of the tile's nibble/3-bit code plane and its
//     sign|mantissa plane;
//   - the tile's escapes (explicit modes) are scattered into a shared-memory
//     bitmap + value array, with every per-escape check of _escape_indices
//     done on the way (position < chunk, index < N, strictly increasing);
//   - per 2 codes one shared-memory "pair LUT" load gives both exponents plus
//     range / sentinel flags; escaped elements take their raw exponent from
//     shared memory (the reference's sparse overwrite, codec.py:477, done in
//     registers so every output byte is written exactly once);
//   - words are rebuilt with byte permutes and written with 256-bit stores.
//   Sentinel mode finds each marked element's escape ordinal with a block scan
//   + decoupled look-back over per-tile mark counts (codec.py:459-467).
// Corruption never faults: every index is bounds-checked, and each failed
// check records its smallest offending ordinal/element in sz_decode_status;
// the host raises CorruptionError in the reference's check order.
#include <cstdlib>
#include <type_traits>
#include "sz_common.cuh"
#include "sz_scan.cuh"

namespace sz {

// K3 (offsets_kernel, chunk-offset scan): sz_scan.cuh

// decode tile: kDecItems 32-byte slots per decode thread
constexpr int kDecItems = 2;
constexpr int kDecSlots = kDecItems * kThreads;        // 512 slots per tile

// ------------------------------------------------------------------ K3s
// Sentinel mode (codec.py:459-467): escapes are marked in-band by the top
// code, so an escape's ordinal is the number of marks before it.  This pass
// counts the marks of every decode tile (codes plane only, 0.5 B/element for
// 4-bit codes); offsets_kernel scans the counts, and the persistent decoder's
// stagers turn each tile's marks into the same bitmap / first-index / value
// staging as explicit mode — no look-back inside the streaming kernel.
template <int CB, int EPV>
__device__ __forceinline__ uint32_t slot_marks(const uint32_t* cw, int nv) {
  // per code: all CB bits set == the sentinel; marks are rare, so test the
  // whole slot first and gather the flag bits only when one is present
  uint32_t t[EPV * CB / 32 + 1];
  uint32_t any = 0;
  if constexpr (CB == 4) {
#pragma unroll
    for (int i = 0; i < EPV / 8; ++i) {
      const uint32_t x = cw[i];
      t[i] = x & (x >> 1) & (x >> 2) & (x >> 3) & 0x11111111u;  // nibble == 15
      any |= t[i];
    }
  } else {
#pragma unroll
    for (int g = 0; g < EPV / 4; ++g) {
      const uint32_t v = group_bits<12>(cw, g);
      const uint32_t f = v & (v >> 1) & (v >> 2) & 0x249u;         // code == 7
      any |= f;
      if (g % 2 == 0) t[g / 2] = f; else t[g / 2] |= f << 16;
    }
  }
  if (!any) return 0u;
  uint32_t mk = 0;
  if constexpr (CB == 4) {
#pragma unroll
    for (int i = 0; i < EPV / 8; ++i) {   // bits 0,4,..,28 -> bits 0..7
      uint32_t u = (t[i] | (t[i] >> 3)) & 0x03030303u;
      u = (u | (u >> 6)) & 0x000F000Fu;
      u = (u | (u >> 12)) & 0xFFu;
      mk |= u << (8 * i);
    }
  } else {
#pragma unroll
    for (int i = 0; i < EPV / 8; ++i) {   // bits 0,3,6,9 (+16) -> bits 0..7
      const uint32_t f = t[i];
      const uint32_t u = (f & 1u) | ((f >> 2) & 2u) | ((f >> 4) & 4u) | ((f >> 6) & 8u) |
                         ((f >> 12) & 16u) | ((f >> 14) & 32u) | ((f >> 16) & 64u) |
                         ((f >> 18) & 128u);
      mk |= u << (8 * i);
    }
  }
  if (nv < EPV) mk &= (1u << nv) - 1u;
  return mk;
}

template <int FMT, int CB>
__global__ void __launch_bounds__(kThreads)
    marks_kernel(const uint8_t* __restrict__ codes, uint64_t n, uint64_t codes_len,
                 uint64_t num_tiles, uint32_t tile_slots, uint32_t* __restrict__ tile_marks,
                 uint32_t* __restrict__ mark_bits) {
  constexpr int EPV = kEpv<FMT>;
  constexpr int CBYTES = EPV * CB / 8;
  constexpr int CWORDS = (CBYTES + 3) / 4;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  // 4-bit codes, whole tile inside the stream: the tile's code plane as
  // 16-byte loads, all in flight at once; a mark is a nibble of all ones, so
  // the count is popc of the nibble-AND (no per-slot mask gather)
  constexpr int kVec = CB == 4 ? kDecSlots * CBYTES / 16 / 32 : 0;  // uint4 per lane
  for (uint64_t t = gw; t < num_tiles; t += nw) {   // one warp per tile
    uint32_t cnt = 0;
    if constexpr (CB == 4) {
      if ((t + 1) * tile_slots * EPV <= n && !(reinterpret_cast<uintptr_t>(codes) & 15)) {
        const uint4* q = reinterpret_cast<const uint4*>(codes + t * tile_slots * CBYTES);
        uint4 v[kVec];
#pragma unroll
        for (int i = 0; i < kVec; ++i) v[i] = __ldg(q + lane + 32 * i);
        // 16 code bytes = 32 elements = one word of the element mark bitmap
        uint32_t* const mb = mark_bits + t * tile_slots * EPV / 32;
#pragma unroll
        for (int i = 0; i < kVec; ++i) {
          const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
          uint32_t word = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t f = w4[k] & (w4[k] >> 1) & (w4[k] >> 2) & (w4[k] >> 3) & 0x11111111u;
            cnt += __popc(f);
            uint32_t u = (f | (f >> 3)) & 0x03030303u;     // nibble flags -> 8 bits
            u = (u | (u >> 6)) & 0x000F000Fu;
            u = (u | (u >> 12)) & 0xFFu;
            word |= u << (8 * k);
          }
          mb[lane + 32 * i] = word;
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
        if (lane == 0) tile_marks[t] = cnt;
        continue;
      }
    }
    for (uint32_t j = lane; j < tile_slots; j += 32) {
      const uint64_t e0 = (t * tile_slots + j) * EPV;
      if (e0 >= n) break;
      const int nv = e0 + EPV <= n ? EPV : static_cast<int>(n - e0);
      uint32_t cw[CWORDS];
      if (nv == EPV && !(CBYTES & 3)) {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(codes + e0 * CB / 8);
#pragma unroll
        for (int i = 0; i < CWORDS; ++i) cw[i] = __ldg(q + i);
      } else {
        ld_bytes_clipped<CBYTES>(codes, e0 * CB / 8, cw, codes_len);
      }
      const uint32_t mk = slot_marks<CB, EPV>(cw, nv);
      cnt += __popc(mk);
      const uint64_t slot_g = t * tile_slots + j;       // EPV-bit field of the bitmap
      if constexpr (EPV == 32) mark_bits[slot_g] = mk;
      else reinterpret_cast<uint16_t*>(mark_bits)[slot_g] = static_cast<uint16_t>(mk);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if (lane == 0) tile_marks[t] = cnt;
  }
}

// ------------------------------------------------------------------ K3a
// abs32 mode: first escape ordinal of every decode tile.  Positions are
// ascending element indices (codec.py:500-507), so ordinal o opens tiles
// (tile(pos[o-1]), tile(pos[o])]; one coalesced pass over the positions
// writes every boundary once (a per-tile binary search would be ~20
// dependent memory latencies).  Unsorted (corrupt) streams leave some
// boundaries at their zeroed value; the decoder clamps, and flags them.
__global__ void __launch_bounds__(kThreads)
    abs_bounds_kernel(const uint32_t* __restrict__ pos, const uint64_t* m_ptr, uint64_t m_host,
                      uint64_t n, uint64_t tile_elems, uint64_t num_tiles,
                      uint64_t* __restrict__ bounds) {
  const uint64_t m = m_ptr ? min(*m_ptr, m_host) : m_host;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t first = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  auto tile_of = [&](uint64_t o) -> uint64_t {  // tile holding ordinal o's element
    const uint64_t t = pos[o] / tile_elems;
    return t < num_tiles ? t : num_tiles;
  };
  for (uint64_t o = first; o <= m; o += stride) {
    const uint64_t t_prev = o == 0 ? 0 : tile_of(o - 1) + 1;  // first tile not before o-1
    const uint64_t t_cur = o == m ? num_tiles : tile_of(o);
    for (uint64_t b = t_prev; b <= t_cur; ++b) bounds[b] = o;
  }
}

template <int POSB>
__device__ __forceinline__ uint64_t load_pos(const void* p, uint64_t o) {
  if constexpr (POSB == 1) return static_cast<const uint8_t*>(p)[o];
  else if constexpr (POSB == 2) return static_cast<const uint16_t*>(p)[o];
  else return static_cast<const uint32_t*>(p)[o];
}

// ------------------------------------------------------------------ K3e
// Escape-dense chunk-relative streams (codec.py:509-536, ε of a few %, e.g.
// top-8 3-bit books at ~7%): the per-ordinal position work moves out of the
// decoder's stagers into a flat pass.  One warp per 16384-element window:
//   - the window's chunk offsets (K3) in shared memory, ordinals in rounds of
//     32 with the next 4 rounds' positions / values in flight, each lane's
//     chunk found from the previous round's (one compare when a round crosses
//     at most one chunk start);
//   - every per-ordinal check of _escape_indices and the value checks
//     (codec.py:451-457, 515-535), first offending ordinal per check;
//   - the window's element escape bitmap built with shared-memory ORs and
//     written once with 16-byte stores, and the escape count of every decode
//     tile in it (popc of its words).
// The decoder then stages a tile exactly like sentinel mode: its bitmap words
// (coalesced), a warp scan for each slot's first compact index, and its
// values as one contiguous run from the scanned tile counts.  Windows are a
// multiple of every decode tile, so every bitmap word and tile count has one
// writer (no atomics in global memory, no zeroing pass).
constexpr int kMarkWin = 16384;
constexpr int kMarkWinWords = kMarkWin / 32;
constexpr int kMarkWarps = 8;
constexpr uint32_t kMarkMinChunk = 32;                        // dense path needs chunk >= 32
constexpr int kMarkMaxChunks = kMarkWin / kMarkMinChunk + 2;  // chunks touching a window, + end

struct MarkArgs {
  const uint64_t* m_ptr;
  uint64_t m;
  const uint64_t* offsets;   // chunk ordinal offsets (K3), n_chunks + 1
  const void* positions;
  const uint8_t* values;
  uint64_t n, n_windows;
  uint64_t n_words;          // bitmap words = decode tiles x tile_words
  uint32_t chunk, tile_words, exp_bins;
  uint32_t esc_ok[8];        // valid escape values (not in the book) as a 256-bit set
  uint32_t* mark_bits;
  uint32_t* tile_marks;
  sz_decode_status* status;
};

struct alignas(16) MarkSmem {
  uint32_t bits[kMarkWinWords];
  uint32_t srel[kMarkMaxChunks];   // chunk starts as ordinals relative to the window's first
};
static_assert(sizeof(MarkSmem) % 16 == 0, "per-warp K3e state stays 16-byte aligned");
static_assert(kMarkWarps * 32 == 256, "one thread per entry of the K3e value table");

template <int POSB>
__global__ void __launch_bounds__(kMarkWarps * 32) escape_marks_kernel(const MarkArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int lane = threadIdx.x & 31;
  MarkSmem& S = reinterpret_cast<MarkSmem*>(smem_raw)[threadIdx.x >> 5];
  __shared__ uint8_t s_vbad[256];     // 1: not a valid escape value (domain or in the book)
  pdl_trigger();
  s_vbad[threadIdx.x] = ((a.esc_ok[threadIdx.x >> 5] >> (threadIdx.x & 31)) & 1u) ^ 1u;
  for (int i = lane; i < kMarkWinWords / 4; i += 32)
    reinterpret_cast<uint4*>(S.bits)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  pdl_wait();
  const uint64_t m = a.m_ptr ? min(*a.m_ptr, a.m) : a.m;
  const uint64_t chunk = a.chunk;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t w = gw; w < a.n_windows; w += nw) {
    const uint64_t e0 = w * kMarkWin, e1 = min(e0 + kMarkWin, a.n);
    const uint64_t ka = e0 / chunk;
    const uint32_t nk = static_cast<uint32_t>((e1 - 1) / chunk - ka + 1);  // chunks in the window
    const uint64_t* const offk = a.offsets + ka;
    const uint64_t o_lo = min(offk[0], m), o_hi = max(min(offk[nk], m), o_lo);
    const uint64_t n_o = o_hi - o_lo;
    // window-relative element of chunk ka's start (<= 0) and the bounds of
    // a hit / of the stream, in 32-bit arithmetic
    const int32_t kbase = static_cast<int32_t>(static_cast<int64_t>(ka * chunk) -
                                               static_cast<int64_t>(e0));
    const uint32_t span = static_cast<uint32_t>(e1 - e0);
    const int32_t past = static_cast<int32_t>(min(a.n - e0, static_cast<uint64_t>(0x7FFFFFFF)));
    if (n_o < (1ull << 31)) {
      // Fast path: the window's chunk starts as u32 ordinals relative to o_lo
      uint32_t* const srel = S.srel;
      for (uint32_t i = lane; i <= nk; i += 32)
        srel[i] = static_cast<uint32_t>(max(min(offk[i], m), o_lo) - o_lo);
      __syncwarp();
      const uint32_t no = static_cast<uint32_t>(n_o);
      using PosT = typename std::conditional<POSB == 1, uint8_t, uint16_t>::type;
      const PosT* const pos_w = static_cast<const PosT*>(a.positions) + o_lo;
      const uint8_t* const val_w = a.values + o_lo;
      const uint32_t chunk32 = a.chunk;
      // Rounds of 32 consecutive ordinals (coalesced loads, the next 4
      // rounds' in flight).  The chunk of each ordinal comes from the
      // warp-uniform starts of the current chunk and the next two (s0, s1,
      // s2 in registers): one compare when a round crosses at most one chunk
      // start, a per-lane search from the current chunk otherwise.  An
      // ordinal is its chunk's first exactly when it equals its chunk's
      // start, which is all the increasing-position check needs besides the
      // predecessor's position.  (A variant staging each lane's contiguous
      // slice in shared memory and walking it with a running chunk index
      // issued fewer loads but measured 2x slower: its per-ordinal branches
      // and the staging stores' load latency.)
      constexpr int U = 4;
      const uint8_t* const vbad = s_vbad;
      uint32_t cur = 0, s0 = 0, s1 = 0, s2 = 0;
      auto refill = [&]() {
        s0 = srel[cur];
        s1 = cur + 1 < nk ? srel[cur + 1] : ~0u;
        s2 = cur + 2 <= nk ? srel[cur + 2] : ~0u;
      };
      refill();
      uint32_t carry_pv = 0;     // position of the previous round's last ordinal
      uint32_t pvs[U], vs[U];
      auto load_batch = [&](uint32_t b0, uint32_t (&pp)[U], uint32_t (&vv)[U]) {
        const PosT* const pb = pos_w + b0 + lane;
        const uint8_t* const vb = val_w + b0 + lane;
        if (b0 + 32 * U <= no) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            pp[u] = static_cast<uint32_t>(pb[32 * u]);
            vv[u] = static_cast<uint32_t>(vb[32 * u]);
          }
        } else {
          const uint32_t left = no - b0 - lane;  // > 32u exactly when ordinal 32u + lane exists
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const bool in = static_cast<int32_t>(left) > 32 * u;
            pp[u] = in ? static_cast<uint32_t>(pb[32 * u]) : 0u;
            vv[u] = in ? static_cast<uint32_t>(vb[32 * u]) : 0u;
          }
        }
      };
      // one round of 32 ordinals; the bitmap OR is unconditional (a lane
      // without a hit ORs 0 into word 0), so the only divergent branch left
      // is the rare failed check
      auto round = [&](uint32_t br, uint32_t pv, uint32_t v) {
        const uint32_t orl = br + lane;
        const bool full = br + 32 <= no;           // warp-uniform
        const uint32_t last = full ? br + 31 : no - 1;
        uint32_t k, sk;
        if (s2 <= last) {                          // warp-uniform: 2+ chunk starts in the round
          uint32_t hi = nk;
          k = cur;
          while (hi - k > 1) {
            const uint32_t mid = (k + hi) >> 1;
            if (srel[mid] <= orl) k = mid; else hi = mid;
          }
          sk = srel[k];
          cur = __shfl_sync(0xffffffffu, k, 31);
          refill();
        } else {
          const bool up = orl >= s1;
          k = cur + (up ? 1u : 0u);
          sk = up ? s1 : s0;
          if (last >= s1) {                        // warp-uniform: the round crosses one start
            ++cur;
            s0 = s1;
            s1 = s2;
            s2 = cur + 2 <= nk ? srel[cur + 2] : ~0u;
          }
        }
        uint32_t prev = __shfl_up_sync(0xffffffffu, pv, 1);
        if (lane == 0) prev = carry_pv;
        carry_pv = __shfl_sync(0xffffffffu, pv, 31);
        const int32_t rel = kbase + static_cast<int32_t>(k * chunk32 + pv);
        const bool live = full || orl < no;
        const bool over = pv >= chunk32, beyond = rel >= past;
        const bool not_inc = orl != sk && prev >= pv;
        // one byte-table test covers the domain and the in-book check
        if (__builtin_expect(live && (vbad[v] | over | beyond | not_inc), 0)) {
          // rare: the reference's checks in order (codec.py:446-536)
          const uint64_t o = o_lo + orl;
          if (v >= a.exp_bins) record_first(&a.status->first_inv[SZ_DEC_VALUE_DOMAIN], o);
          else if (vbad[v]) record_first(&a.status->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
          if (over) record_first(&a.status->first_inv[SZ_DEC_POS_OVER_CHUNK], o);
          else if (beyond) record_first(&a.status->first_inv[SZ_DEC_POS_PAST_END], o);
          else if (not_inc) record_first(&a.status->first_inv[SZ_DEC_POS_NOT_INC], o);
        }
        const bool hit = live && !over && static_cast<uint32_t>(rel) < span;
        const uint32_t ur = hit ? static_cast<uint32_t>(rel) : 0u;
        atomicOr(&S.bits[ur >> 5], hit ? 1u << (ur & 31) : 0u);
      };
      // ping-pong batches: the next batch's loads land in the other register
      // set while this one is processed (no register copies)
      uint32_t qpvs[U], qvs[U];
      if (no) load_batch(0, pvs, vs);
      for (uint32_t b0 = 0; b0 < no; b0 += 64 * U) {
        if (b0 + 32 * U < no) load_batch(b0 + 32 * U, qpvs, qvs);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (b0 + 32 * u < no) round(b0 + 32 * u, pvs[u], vs[u]);
        if (b0 + 32 * U >= no) break;
        if (b0 + 64 * U < no) load_batch(b0 + 64 * U, pvs, vs);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (b0 + 32 * (U + u) < no) round(b0 + 32 * (U + u), qpvs[u], qvs[u]);
      }
    } else {
      // corrupt counts (> 2^31 ordinals in one window): plain per-ordinal
      // loop in 64-bit arithmetic, same checks
      for (uint64_t o = o_lo + lane; o < o_hi; o += 32) {
        uint32_t lo = 0, hi = nk;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (min(offk[mid], m) <= o) lo = mid; else hi = mid;
        }
        const uint32_t pv = static_cast<uint32_t>(load_pos<POSB>(a.positions, o));
        const uint32_t v = a.values[o];
        const uint64_t idx = (ka + lo) * chunk + pv;
        const bool in_book = s_vbad[v];   // (after the domain check)
        if (v >= a.exp_bins) record_first(&a.status->first_inv[SZ_DEC_VALUE_DOMAIN], o);
        else if (in_book) record_first(&a.status->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
        if (pv >= chunk) {
          record_first(&a.status->first_inv[SZ_DEC_POS_OVER_CHUNK], o);
        } else if (idx >= a.n) {
          record_first(&a.status->first_inv[SZ_DEC_POS_PAST_END], o);
        } else {
          if (o > min(offk[lo], m) && static_cast<uint32_t>(load_pos<POSB>(a.positions, o - 1)) >= pv)
            record_first(&a.status->first_inv[SZ_DEC_POS_NOT_INC], o);
          if (idx >= e0 && idx < e1) {
            const uint32_t r = static_cast<uint32_t>(idx - e0);
            atomicOr(&S.bits[r >> 5], 1u << (r & 31));
          }
        }
      }
    }
    __syncwarp();
    // flush: 16-byte stores of the window's words, each decode tile's count,
    // and the shared words zeroed for the next window
    const uint64_t wd0 = e0 / 32;
    const uint32_t pieces_per_tile = a.tile_words / 128;   // 128 words per round of 32 lanes
    uint32_t tsum = 0;
#pragma unroll
    for (int j = 0; j < kMarkWinWords / 128; ++j) {
      uint4* sq = reinterpret_cast<uint4*>(S.bits) + lane + 32 * j;
      const uint4 q = *sq;
      *sq = make_uint4(0, 0, 0, 0);
      const uint64_t wd = wd0 + 4ull * (lane + 32 * j);
      if (wd + 4 <= a.n_words) *reinterpret_cast<uint4*>(a.mark_bits + wd) = q;
      tsum += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
      if ((j + 1) % pieces_per_tile == 0) {  // one warp sum per decode tile
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, d);
        const uint64_t tile = (wd0 + 128ull * (j + 1) - 1) / a.tile_words;
        if (lane == 0 && tile * a.tile_words < a.n_words) a.tile_marks[tile] = tsum;
        tsum = 0;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K4
struct DecodeArgs {
  const uint64_t* m_ptr;     // optional device-resident M
  const uint8_t* codes;
  const uint8_t* sm;
  const uint64_t* offsets;   // chunked mode
  const void* positions;
  const uint8_t* values;
  uint64_t n, m;
  uint8_t* out;
  sz_decode_status* status;
  uint64_t* states;          // sentinel look-back
  unsigned long long* tile_counter;
  uint64_t num_tiles;
  uint64_t n_chunks;
  uint64_t codes_len, sm_len;
  uint32_t chunk;
  int32_t chunk_shift;
  // Segmented (paged) output: when non-null, element
  // byte offset o of the stream lands at seg_addrs[o >> seg_shift] + (o & mask)
  // — decoded words go straight into the destination's KV-cache blocks.
  const uint64_t* seg_addrs;
  uint32_t seg_shift;
  const uint32_t* mark_bits;  // sentinel: element mark bitmap from K3s
};

// Address of the 32-byte output slot starting at element e0 (slots never
// straddle segments: segments are >= 32 bytes, powers of two).
template <int WB>
__device__ __forceinline__ uint8_t* out_slot(const DecodeArgs& a, uint64_t e0) {
  if (!a.seg_addrs) return a.out + e0 * WB;
  const uint64_t o = e0 * WB;
  return reinterpret_cast<uint8_t*>(__ldg(a.seg_addrs + (o >> a.seg_shift))) +
         (o & ((1ull << a.seg_shift) - 1));
}

template <int NBYTES>
__device__ __forceinline__ void ld_packed(const uint8_t* src, uint32_t* w) {
  if constexpr (NBYTES == 16) {
    const uint4 v = ld_stream128(src);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else if constexpr (NBYTES == 12) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    w[0] = __ldg(s); w[1] = __ldg(s + 1); w[2] = __ldg(s + 2);
  } else if constexpr (NBYTES == 8) {
    const uint2 v = ld_stream64(src);
    w[0] = v.x; w[1] = v.y;
  } else if constexpr (NBYTES == 6) {
    const uint16_t* s = reinterpret_cast<const uint16_t*>(src);
    w[0] = __ldg(s) | (static_cast<uint32_t>(__ldg(s + 1)) << 16);
    w[1] = __ldg(s + 2);
  }
}

template <int FMT>
__device__ __forceinline__ void rebuild_group(uint32_t e4, uint32_t a4, uint32_t* outw, int g) {
  if constexpr (FMT == SZ_BF16) {
    const uint32_t lo4 = (a4 & 0x7F7F7F7Fu) | ((e4 << 7) & 0x80808080u);
    const uint32_t hi4 = (a4 & 0x80808080u) | ((e4 >> 1) & 0x7F7F7F7Fu);
    outw[2 * g] = __byte_perm(lo4, hi4, 0x5140);
    outw[2 * g + 1] = __byte_perm(lo4, hi4, 0x7362);
  } else if constexpr (FMT == SZ_E5M2) {
    outw[g] = ((a4 << 5) & 0x80808080u) | (e4 << 2) | (a4 & 0x03030303u);
  } else {
    outw[g] = ((a4 << 4) & 0x80808080u) | (e4 << 3) | (a4 & 0x07070707u);
  }
}

// E5M2 12-bit sign|mantissa group (four 3-bit symbols a = s<<2 | m,
// formats.py:123-125,184-189) -> the sign and mantissa bits of four E5M2
// bytes (bit 7 and bits 0-1).  The two spreads and the final a*33 (copies
// bit 2 of each symbol to bit 7) are left shifts the compiler can issue on
// the FMA pipe, next to the ALU-bound lookups.
__device__ __forceinline__ uint32_t e5m2_sm_bytes(uint32_t v12) {
  const uint32_t u = (v12 | (v12 << 10)) & 0x003F003Fu;  // symbols (0,1) | (2,3) << 16
  const uint32_t t = (u | (u << 5)) & 0x07070707u;       // one symbol per byte
  return (t * 33u) & 0x83838383u;
}

// Escape values staged per tile, compact in ordinal order (the decode warp
// finds a value as slot_first[slot] + rank within the slot's bitmap word);
// tiles with more escapes read the rest straight from global memory.
// E5M2 tiles hold 16384 elements: 2048 values cover escape-dense books
// (7% of a tile); E4M3's larger sign|mantissa plane leaves no room for it.
template <int FMT> constexpr int kDecValCap = FMT == SZ_E5M2 ? 2048 : 1024;
constexpr uint32_t kNoEscape = 0xFFFFFFFFu;

// Value of escape bit j of a slot: compact index = the slot's first index +
// rank of bit j among the slot's escape bits (valid streams have ascending
// ordinals in element order); beyond the staged capacity read global memory.
// Corrupt streams (flagged elsewhere) only ever get a bounded read.
template <int CAP>
__device__ __forceinline__ uint32_t escape_value(const uint8_t* vals, uint32_t first,
                                                 uint32_t bm0, int j, uint64_t ofirst,
                                                 uint64_t m, const uint8_t* gvals) {
  const uint64_t c = static_cast<uint64_t>(first) + __popc(bm0 & ((1u << j) - 1u));
  if (c < static_cast<uint64_t>(CAP)) return vals[c];
  return ofirst + c < m ? gvals[ofirst + c] : 0u;
}

// Escape overwrite of one 4-element group without a per-escape loop.  The
// group's escape bits mg (4 bits) select, through one PRMT, bytes of the
// 4-byte window of staged values starting at the group's first rank r
// (values are compact in element order) in place of the dense exponent
// bytes: selector nibble k = rank of element k among the group's escapes
// when bit k is set, else 4 + k (keep).  The selectors of all 16 patterns
// sit in shared memory.  Explicit modes also check the escaped elements'
// dense codes (codec.py:472-476): an in-range code is 0 exactly when its
// exponent is the book's first entry (entries are distinct; out-of-range
// codes are CODE_RANGE, an earlier check).  Returns the updated bytes;
// *nondummy gets the mask of escaped bytes whose exponent is not entry 0.
__device__ __forceinline__ uint32_t merge_group(uint32_t e4, uint32_t mg, uint32_t r,
                                                uint32_t vals_base, uint32_t sel_base,
                                                uint32_t keep4, uint32_t* nondummy) {
  const uint32_t sel = lds_u32(sel_base + 4 * mg);
  const uint32_t ad = vals_base + r;    // (vals_base need not be word aligned)
  const uint32_t a0 = ad & ~3u;
  const uint32_t v4 = __funnelshift_r(lds_u32(a0), lds_u32(a0 + 4), 8 * (ad & 3));
  *nondummy = (e4 ^ keep4) & __byte_perm(0xFFFFFFFFu, 0u, sel);
  return __byte_perm(v4, e4, sel);
}

// First escaped element of a slot whose dense code is not the dummy code 0
// (codec.py:472-476), recorded in the status; called only when the
// group-wise merge saw one (corrupt streams).
template <int CB, int CWORDS>
__device__ __forceinline__ void first_nondummy(const uint32_t* cw, uint32_t bm, uint64_t e0,
                                               sz_decode_status* st) {
  while (bm) {
    const int j = __ffs(bm) - 1;
    bm &= bm - 1;
    const int bit = CB * j;
    const uint64_t lo = pick<CWORDS>(cw, bit >> 5);
    const uint64_t hi = (bit >> 5) + 1 < CWORDS ? pick<CWORDS>(cw, (bit >> 5) + 1) : 0u;
    const uint32_t code = static_cast<uint32_t>(((hi << 32) | lo) >> (bit & 31)) & ((1u << CB) - 1);
    if (code != 0) {
      record_first(&st->first_inv[SZ_DEC_NONDUMMY], e0 + j);
      return;
    }
  }
}

// ------------------------------------------------------------------ K4 (persistent)
// Explicit modes (chunk-relative and abs32).  Same warp-specialised shape as
// the encoder: warp 8 streams each tile's code and sign|mantissa planes into a
// shared-memory ring with TMA bulk copies; warp 9 stages the tile's escapes
// (bitmap + raw values in smem) and runs every per-escape check; warps 0-7
// decode slots from smem and write 256-bit stores.  No CTA-wide barriers in
// steady state — only mbarrier hand-offs.
constexpr int kDecHelpers = 3;                          // escape-staging warps
constexpr int kPosMarked = 8;   // K4 POSB of escape-dense chunk-relative streams (K3e)
constexpr int kDecThreads = kThreads + 32 * (1 + kDecHelpers);
constexpr int kDecOffStage = 64;                        // staged chunk offsets per helper
template <int FMT, int NSTAGES = 5, int CB = 4>
struct DecSmem {
  static constexpr int STAGES = NSTAGES;
  static constexpr int EPV = kEpv<FMT>;
  static constexpr int TILE = kDecSlots * EPV;
  alignas(128) uint8_t codes[STAGES][TILE * CB / 8];
  alignas(128) uint8_t sm[STAGES][TILE * Fmt<FMT>::kSmBits / 8];
  uint32_t bitmap[STAGES][TILE / 32];
  uint32_t slot_first[STAGES][kDecSlots];  // compact index of a slot's first escape
  // escape values by (ordinal - ofirst), from byte vshift (< 16: the K3e
  // stager keeps the run's 16-byte quads at their global alignment); 8
  // bytes of slack for the decode warps' 4-byte window reads (merge_group)
  // at the end of the run
  alignas(16) uint8_t vals[STAGES][kDecValCap<FMT> + 32];
  uint64_t ofirst[STAGES];                 // ordinal of the tile's first escape
  uint32_t vshift[STAGES];
  uint64_t off[kDecHelpers][kDecOffStage + 1];
  uint64_t meta[STAGES];
  uint64_t full[STAGES];
  uint64_t staged[STAGES];
  uint64_t claimed[STAGES];   // producer -> stagers: tile id written (before TMA)
  uint64_t empty[STAGES];
};

// CTAs per SM and ring depth.  The K3e instantiation and every E5M2 decoder
// run 3 CTAs per SM (24 decode warps instead of 16) on a shallower ring — 4
// stages (BF16) / 3 (FP8) keep 3 CTAs' shared memory within the SM, 56
// registers the file: the K3e merge is latency-bound (BF16 top-8 3-bit
// 2016 -> 2059 GB/s) and so is E5M2's decode (c3 2925 -> 2999 GB/s,
// alternating A/B runs on one box).  Realistic BF16 keeps 2 x 5 stages (it
// runs at the copy peak).
// K3e instantiation with 3-bit codes: one 4096-entry table maps a 12-bit
// code group straight to its four exponent bytes (16 KiB of shared memory;
// its ring drops to 3 stages so 3 CTAs still fit an SM): one lookup per 4
// elements instead of two pair lookups, their address arithmetic and a
// PRMT — top-8 3-bit decode BF16 2067 -> 2095, E5M2 1196 -> 1297 GB/s.
// FP8 decoders on the position paths (3 CTAs x 3 stages) use it too.
#ifdef SZ_NO_T12_FP8
constexpr bool kT12Fp8 = false;
#else
constexpr bool kT12Fp8 = true;
#endif
template <int CB, int PMODE, int FMT = SZ_BF16>
constexpr bool kT12 = CB == 3 && (PMODE == kPosMarked ||
                                  (kT12Fp8 && FMT != SZ_BF16 && PMODE != 0));
// E4M3 decodes like E5M2 (one byte per element, twice BF16's elements per
// byte of traffic): 3 CTAs per SM on a 3-stage ring.
#ifdef SZ_E4_2CTA
constexpr bool kFp8ThreeCtas = false;
#else
constexpr bool kFp8ThreeCtas = true;
#endif
template <int FMT>
constexpr bool kDec3Ctas = FMT == SZ_E5M2 || (FMT == SZ_E4M3 && kFp8ThreeCtas);
template <int FMT, int CB, int PMODE>
constexpr int kDecStages = PMODE == kPosMarked ? (FMT == SZ_BF16 && !kT12<CB, PMODE> ? 4 : 3)
                                               : (kDec3Ctas<FMT> ? 3 : 5);
template <int FMT, int PMODE>
constexpr int kDecCtasPerSm = PMODE == kPosMarked || kDec3Ctas<FMT> ? 3 : 2;

template <int FMT, int CB, int PMODE>
__global__ void __launch_bounds__(kDecThreads, kDecCtasPerSm<FMT, PMODE>)
    decode_persistent(const __grid_constant__ sz_params p, const DecodeArgs a) {
  // PMODE = position bytes (1, 2, 4 abs32), 0 sentinel, kPosMarked (K3e)
  constexpr int POSB = PMODE;
  constexpr int EPV = kEpv<FMT>;
  constexpr int G = EPV / 4;
  constexpr int WB = Fmt<FMT>::kWordBytes;
  constexpr int SMB = Fmt<FMT>::kSmBits;
  constexpr int CBYTES = EPV * CB / 8;
  constexpr int SBYTES = EPV * SMB / 8;
  constexpr int CWORDS = (CBYTES + 3) / 4;
  constexpr int SWORDS = (SBYTES + 3) / 4;
  constexpr uint64_t TILE = static_cast<uint64_t>(kDecSlots) * EPV;
  constexpr bool ABS = POSB == 4;
  constexpr bool SENT = POSB == 0;   // sentinel mode: marks in the code plane
  // escape bitmap + tile ordinal bases from a pre-pass: K3s (sentinel) or
  // K3e (escape-dense chunk-relative streams, POSB == kPosMarked)
  constexpr bool MARKED = SENT || POSB == kPosMarked;
  // escape-dense streams (the K3e path): escapes merged group by group
  // (merge_group) instead of the per-escape loop, which serialises a warp
  // on its densest slot; sparse streams keep the loop (smaller code, ~1
  // escape per warp round)
  constexpr bool kGroupMerge = POSB == kPosMarked;
  constexpr int LUT2 = CB == 4 ? 256 : 64;
  constexpr uint32_t kCodeMask = (1u << CB) - 1;
  using Smem = DecSmem<FMT, kDecStages<FMT, CB, PMODE>, CB>;
  constexpr int kStages = Smem::STAGES;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_trigger();
  // Pair LUT in static shared memory, 1 KiB aligned: the address of entry i
  // is base | (i << 2), formed with one SHF + one LOP3 (no base add).
  __shared__ __align__(1024) uint32_t s_lut2[256];
  for (int i = tid; i < LUT2; i += kDecThreads) {
    const uint32_t c0 = i & kCodeMask, c1 = (i >> CB) & kCodeMask;
    const uint32_t bad = (c0 >= p.n_entries) | ((c1 >= p.n_entries) << 1);
    s_lut2[i] = p.dec_lut[c0] | (p.dec_lut[c1] << 8) | (bad << 16);
  }
  const uint32_t lut2_base = smem_addr(s_lut2);
  constexpr bool T12 = kT12<CB, PMODE, FMT>;
  __shared__ __align__(16) uint32_t s_t12[T12 ? 4096 : 1];
  if constexpr (T12) {
    for (int i = tid; i < 4096; i += kDecThreads)
      s_t12[i] = p.dec_lut[i & 7] | (p.dec_lut[(i >> 3) & 7] << 8) |
                 (p.dec_lut[(i >> 6) & 7] << 16) | (p.dec_lut[i >> 9] << 24);
  }
  const uint32_t t12_base = smem_addr(s_t12);
  // In-book exponents as a 256-bit set in shared memory: the stagers' value
  // checks index it by escape value (a divergent index into the kernel
  // parameters' enc_lut would serialise the constant cache per distinct value).
  __shared__ uint32_t s_inbook[8];
  if (tid < 8) {
    uint32_t w = 0;
    for (int b = 0; b < 32; ++b) w |= ((p.enc_lut[tid * 32 + b] >> 4) & 1u) << b;
    s_inbook[tid] = w;
  }
  auto in_book = [&](uint32_t v) { return (s_inbook[v >> 5] >> (v & 31)) & 1u; };
  // merge_group's PRMT selectors, one per 4-bit escape pattern
  __shared__ uint32_t s_sel[16];
  if (tid < 16) {
    uint32_t sel = 0, rank = 0;
    for (int k = 0; k < 4; ++k) {
      const uint32_t nib = (tid >> k) & 1 ? rank++ : 4u + k;
      sel |= nib << (4 * k);
    }
    s_sel[tid] = sel;
  }
  const uint32_t sel_base = smem_addr(s_sel);
  const uint32_t d0 = p.dec_lut[0];   // exponent of dense code 0 (the dummy)
  // E5M2 with 4-bit codes: a pair table indexed by a code byte (elements
  // 2i, 2i+1) whose u16 entries hold both exponents already at their E5M2
  // bit positions (bits 2-6 of each byte) — reconstruct (formats.py:136-155)
  // becomes two lookups, one byte permute and the sign-mantissa bits.
  constexpr bool kE5Fast = FMT == SZ_E5M2 && CB == 4;
  __shared__ __align__(1024) uint16_t s_e5[kE5Fast ? 256 : 2];
  const uint8_t* e5tab = reinterpret_cast<const uint8_t*>(s_e5);
  if constexpr (kE5Fast) {
    for (int b = tid; b < 256; b += kDecThreads)
      s_e5[b] = static_cast<uint16_t>((p.dec_lut[b & 15] << 2) | (p.dec_lut[b >> 4] << 10));
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.staged[s], 32);  // every stager lane arrives
      mbar_init(&S.claimed[s], 1);
      mbar_init(&S.empty[s], kThreads);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // the shared-memory prologue above only reads kernel parameters; from here
  // on the predecessor grid's results are read
  pdl_wait();
  const uint64_t n = a.n, m = a.m_ptr ? min(*a.m_ptr, a.m) : a.m;
  if (a.m_ptr && blockIdx.x == 0 && tid == 0 && *a.m_ptr > a.m)
    atomicOr(&a.status->flags, 1u << SZ_DEC_CAPACITY);

  if (warp == kWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const uint32_t s = it % kStages, ph = (it / kStages) & 1;
        mbar_wait(&S.empty[s], ph ^ 1);
        const uint64_t tile = atomicAdd(a.tile_counter, 1ull);
        if (tile >= a.num_tiles) {
          // end markers: this iteration (decode warps) and one per helper
          for (uint32_t k = 0; k < kDecHelpers; ++k) {
            const uint32_t sk = (it + k) % kStages, pk = ((it + k) / kStages) & 1;
            if (k) mbar_wait(&S.empty[sk], pk ^ 1);
            S.meta[sk] = ~0ull;
            mbar_arrive(&S.claimed[sk]);
            mbar_arrive(&S.full[sk]);
          }
          break;
        }
        S.meta[s] = tile;
        // stagers start on the tile's escapes while its planes are in flight
        mbar_arrive(&S.claimed[s]);
        const uint64_t e0 = tile * TILE;
        const uint32_t full_slots = static_cast<uint32_t>(min(n - e0, TILE) / EPV);
        const uint32_t cbytes = (full_slots * CBYTES) & ~15u;
        const uint32_t sbytes = (full_slots * SBYTES) & ~15u;
        mbar_arrive_tx(&S.full[s], cbytes + sbytes);
        if (cbytes) tma_load_1d(S.codes[s], a.codes + e0 * CB / 8, cbytes, &S.full[s]);
        if (sbytes) tma_load_1d(S.sm[s], a.sm + e0 * SMB / 8, sbytes, &S.full[s]);
      }
    }
    return;
  }

  if (warp > kWarps) {
    // ------------------------------------------------------------ escape stagers
    // kDecHelpers warps, helper h owns iterations it == h (mod kDecHelpers), so
    // the dependent global loads of several tiles are in flight at once.
    const uint32_t exp_bins = 1u << Fmt<FMT>::kExpBits;
    const int h = warp - kWarps - 1;
    uint64_t* soff = S.off[h];
    for (uint32_t it = h;; it += kDecHelpers) {
      const uint32_t s = it % kStages, ph = (it / kStages) & 1;
      mbar_wait(&S.claimed[s], ph);
      const uint64_t tile = S.meta[s];
      if (tile == ~0ull) break;
      const uint64_t s0 = tile * TILE, s1 = min(s0 + TILE, n);
      // Direct happens-before with the decode warps' last use of this stage
      // (already guaranteed through the producer's chain; free to re-check).
      mbar_wait(&S.empty[s], ph ^ 1);
      if constexpr (!MARKED) {  // (marked staging writes every bitmap word itself)
#pragma unroll
        for (int i = lane; i < static_cast<int>(TILE / 32); i += 32) S.bitmap[s][i] = 0;
#pragma unroll
        for (int i = lane; i < kDecSlots; i += 32) S.slot_first[s][i] = kNoEscape;
      }
      // Stage one in-tile escape: bitmap bit, slot's first compact index,
      // compact value (c = ordinal - first in-tile ordinal).
      auto stage = [&](uint64_t idx, uint64_t c, uint32_t v) {
        const uint32_t rel = static_cast<uint32_t>(idx - s0);
        atomicOr(&S.bitmap[s][rel >> 5], 1u << (rel & 31));
        atomicMin(&S.slot_first[s][rel / EPV], static_cast<uint32_t>(min(c, static_cast<uint64_t>(0xFFFFFFFEu))));
        if (c < kDecValCap<FMT>) S.vals[s][c] = static_cast<uint8_t>(v);
      };
      uint64_t o_first = 0;
      uint32_t vshift = 0;
      if constexpr (ABS) {
        // abs32: per-ordinal checks spread evenly over tiles (the staging
        // below only visits ordinals whose positions land in some tile)
        const uint64_t q = (m + a.num_tiles - 1) / a.num_tiles;
        const uint64_t o0 = tile * q, o1 = min(o0 + q, m);
        const uint32_t* pos = static_cast<const uint32_t*>(a.positions);
        for (uint64_t o = o0 + lane; o < o1; o += 32) {
          const uint32_t v = a.values[o];
          if (v >= exp_bins) record_first(&a.status->first_inv[SZ_DEC_VALUE_DOMAIN], o);
          else if (!in_book(v))
            record_first(&a.status->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
          const uint32_t pv = pos[o];
          if (pv >= n) record_first(&a.status->first_inv[SZ_DEC_ABS_PAST_END], o);
          if (o > 0 && pv <= pos[o - 1]) record_first(&a.status->first_inv[SZ_DEC_ABS_NOT_INC], o);
        }
      }
      if (tile == a.num_tiles - 1 && lane == 0) {
        const uint32_t cbits = static_cast<uint32_t>((n * CB) & 7);
        if (cbits && (a.codes[a.codes_len - 1] >> cbits))
          record_first(&a.status->first_inv[SZ_DEC_CODE_PAD], 0);
        if constexpr (SMB != 8) {
          const uint32_t sbits = static_cast<uint32_t>((n * SMB) & 7);
          if (sbits && (a.sm[a.sm_len - 1] >> sbits))
            record_first(&a.status->first_inv[SZ_DEC_SM_PAD], 0);
        }
      }
      __syncwarp();
      if constexpr (MARKED) {
        // Sentinel mode (codec.py:459-467): the tile's marks come from K3s's
        // scan of its code plane; escape-dense chunk-relative mode: from
        // K3e's walk over the positions.  Its first ordinal is the scan of
        // the per-tile counts.
        const uint64_t t_first = a.offsets[tile];
        const uint64_t t_end = max(a.offsets[tile + 1], t_first);
        o_first = t_first;
        // The tile's marks come as K3s's element bitmap, loaded here right at
        // the claim (no wait for the code plane's TMA): lane-contiguous words,
        // one warp scan for the slots' first compact indices.
        constexpr int SPL = kDecSlots / 32;      // consecutive slots per lane
        constexpr int WPL = SPL * EPV / 32;      // their bitmap words
        const uint4* mb = reinterpret_cast<const uint4*>(a.mark_bits + tile * (TILE / 32) +
                                                         lane * WPL);
        uint32_t wv[WPL];
#pragma unroll
        for (int i = 0; i < WPL / 4; ++i) {
          const uint4 q = __ldg(mb + i);
          wv[4 * i] = q.x; wv[4 * i + 1] = q.y; wv[4 * i + 2] = q.z; wv[4 * i + 3] = q.w;
        }
        const uint64_t valid = s1 - s0;          // elements of the (tail) tile
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
          const uint64_t b0 = static_cast<uint64_t>(lane * WPL + k) * 32;
          if (b0 + 32 > valid) wv[k] = b0 >= valid ? 0u : wv[k] & ((1u << (valid - b0)) - 1u);
        }
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < WPL; ++k) cnt += __popc(wv[k]);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += o;
        }
        uint32_t run = incl - cnt;
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
          const uint32_t slot = lane * SPL + j;
          const uint32_t mk = EPV == 32 ? wv[j] : (wv[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
          if (mk) S.slot_first[s][slot] = run;
          run += __popc(mk);
        }
#pragma unroll
        for (int k = 0; k < WPL; ++k) S.bitmap[s][lane * WPL + k] = wv[k];
        if constexpr (!SENT) {
          // K3e checked every value already: a plain copy of the tile's run.
          // Its 16-byte-aligned interior (<= kDecValCap / 16 quads) is loaded
          // with every load in flight at once — one memory latency after
          // t_first instead of one per 32 words — and the < 16-byte head and
          // tail by single lanes.
          const uint64_t o_hi = min(min(t_end, m), t_first + kDecValCap<FMT>);
          const uintptr_t vb = reinterpret_cast<uintptr_t>(a.values);
          const uint64_t q_lo = (vb + t_first + 15) >> 4, q_hi = (vb + o_hi) >> 4;
          if (o_hi > t_first && q_lo < q_hi) {
            constexpr int kQPL = (kDecValCap<FMT> / 16 + 31) / 32;
            const uint4* qp = reinterpret_cast<const uint4*>(q_lo << 4);
            const uint32_t nq = static_cast<uint32_t>(q_hi - q_lo);
            uint4 qv[kQPL];
#pragma unroll
            for (int j = 0; j < kQPL; ++j)
              if (lane + 32u * j < nq) qv[j] = __ldg(qp + lane + 32 * j);
            const uint64_t head_end = (q_lo << 4) - vb, tail_beg = (q_hi << 4) - vb;
            const uint64_t eo = lane < 16 ? t_first + lane : tail_beg + (lane - 16);
            const bool edge = lane < 16 ? eo < head_end : eo < o_hi;
            const uint8_t eb = edge ? a.values[eo] : 0;
            // staged from byte vshift = the run's global address mod 16, so
            // every interior quad is one aligned 16-byte store
            vshift = static_cast<uint32_t>((vb + t_first) & 15);
            uint8_t* const dv = S.vals[s] + vshift;
            const uint32_t c0 = static_cast<uint32_t>(head_end - t_first);
#pragma unroll
            for (int j = 0; j < kQPL; ++j)
              if (lane + 32u * j < nq)
                *reinterpret_cast<uint4*>(dv + c0 + 16u * (lane + 32u * j)) = qv[j];
            if (edge) dv[eo - t_first] = eb;
          } else {
            for (uint64_t o = t_first + lane; o < o_hi; o += 32) S.vals[s][o - t_first] = a.values[o];
          }
        } else {
          // the tile's values first — staged (first kDecValCap) and checked
          // (codec.py:446-457) for every ordinal its marks reach — while its
          // code plane is still in flight
          const uint64_t o_hi = min(t_end, m);
          for (uint64_t o = t_first + lane; o < o_hi; o += 32) {
            const uint32_t v = a.values[o];
            if (v >= exp_bins) record_first(&a.status->first_inv[SZ_DEC_VALUE_DOMAIN], o);
            else if (!in_book(v))
              record_first(&a.status->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
            if (o - t_first < kDecValCap<FMT>) S.vals[s][o - t_first] = static_cast<uint8_t>(v);
          }
        }
      } else if constexpr (ABS) {
        // the tile's ordinal range from K3a (abs_bounds_kernel); clamped,
        // so a corrupt (unsorted) stream only ever costs bounded reads
        const uint32_t* pos = static_cast<const uint32_t*>(a.positions);
        const uint64_t lo = min(a.offsets[tile], m);
        const uint64_t hi = max(lo, min(a.offsets[tile + 1], m));
        o_first = lo;
        for (uint64_t o = lo + lane; o < hi; o += 32) {
          const uint64_t idx = pos[o];
          if (idx >= s0 && idx < s1) stage(idx, o - lo, a.values[o]);
        }
      } else {
        const uint64_t ka = s0 / a.chunk, kb = (s1 - 1) / a.chunk;
        const uint64_t nk = kb - ka + 2;
        const bool staged = nk <= kDecOffStage + 1;
        if (staged)
          for (uint64_t i = lane; i < nk; i += 32) soff[i] = a.offsets[ka + i];
        __syncwarp();
        const uint64_t* off = staged ? soff : a.offsets + ka;
        const uint64_t o_lo = min(off[0], m), o_hi = min(off[nk - 1], m);
        // 32 consecutive ordinals per round: coalesced position/value loads,
        // the predecessor's position comes from the neighbouring lane.
        uint64_t carry = 0;  // position of ordinal base-1 (previous round's lane 31)
        bool have_first = false;
        // One ordinal per lane per round; escape-heavy ranges keep 4 x 32
        // ordinals per round in flight (all loads before the first use), the
        // common sparse case stays at one short round.
        auto one = [&](uint64_t rbase, uint64_t pv, uint32_t v) {
          const uint64_t o = rbase + lane;
          const bool live = o < o_hi;
          uint64_t prev = __shfl_up_sync(0xffffffffu, pv, 1);
          if (lane == 0) prev = carry;
          carry = __shfl_sync(0xffffffffu, pv, 31);
          uint64_t idx = 0;
          bool hit = false;
          if (live) {
            // per-ordinal value checks (codec.py:451-457); complete coverage when
            // sum(counts) != M is restored on the host (sz_check_values)
            if (v >= exp_bins) record_first(&a.status->first_inv[SZ_DEC_VALUE_DOMAIN], o);
            else if (!in_book(v))
              record_first(&a.status->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
            uint64_t lo = 0, hi = nk - 1;
            while (hi - lo > 1) {
              const uint64_t mid = (lo + hi) >> 1;
              if (off[mid] <= o) lo = mid; else hi = mid;
            }
            idx = (ka + lo) * a.chunk + pv;
            if (pv >= a.chunk) {
              record_first(&a.status->first_inv[SZ_DEC_POS_OVER_CHUNK], o);
            } else if (idx >= n) {
              record_first(&a.status->first_inv[SZ_DEC_POS_PAST_END], o);
            } else {
              if (o > off[lo] && prev >= pv)
                record_first(&a.status->first_inv[SZ_DEC_POS_NOT_INC], o);
              hit = idx >= s0 && idx < s1;
            }
          }
          // the tile's escapes are a contiguous ordinal run (valid streams):
          // its first ordinal anchors the compact value indices
          const uint32_t hb = __ballot_sync(0xffffffffu, hit);
          if (!have_first && hb) {
            o_first = rbase + (__ffs(hb) - 1);
            have_first = true;
          }
          if (hit && o >= o_first) stage(idx, o - o_first, v);
        };
        constexpr int U = 4;
        const uint64_t n_o = o_hi - o_lo;
        if (staged && n_o < (1ull << 31)) {
          // Fast path: the tile's chunk starts as u32 ordinals relative to o_lo
          // (in place of the staged u64 offsets), and each round finds its
          // lanes' chunks from the previous round's: one broadcast compare
          // when the round crosses at most one chunk start (escape-dense
          // tiles), a short binary search otherwise.  All per-ordinal checks
          // fold into one predicate; the rare failing ordinal takes the
          // detailed path.
          uint32_t* const srel = reinterpret_cast<uint32_t*>(soff);
          // in place, 32 entries at a time: block j's u32 stores only overwrite
          // u64 entries < 32j + 16, all read already
          for (uint32_t j0 = 0; j0 < nk; j0 += 32) {
            const uint32_t i = j0 + lane;
            const uint64_t v = i < nk ? soff[i] : 0;
            __syncwarp();
            if (i < nk) srel[i] = static_cast<uint32_t>(min(v, m) - o_lo);
            __syncwarp();
          }
          const uint32_t nch = static_cast<uint32_t>(nk - 1), no = static_cast<uint32_t>(n_o);
          uint32_t cur = 0;  // srel[cur] <= the round's first ordinal
          // batch b + 1's loads are issued before batch b is processed: one
          // exposed memory latency per tile, not one per 4 x 32 ordinals
          uint32_t pvs[U], vs[U];
          auto load_batch = [&](uint32_t b0, uint32_t (&pp)[U], uint32_t (&vv)[U]) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t orl = b0 + 32 * u + lane;
              pp[u] = orl < no ? static_cast<uint32_t>(load_pos<POSB>(a.positions, o_lo + orl)) : 0u;
              vv[u] = orl < no ? a.values[o_lo + orl] : 0u;
            }
          };
          load_batch(0, pvs, vs);
          for (uint32_t b0 = 0; b0 < no; b0 += 32 * U) {
            uint32_t npvs[U], nvs[U];
            if (b0 + 32 * U < no) load_batch(b0 + 32 * U, npvs, nvs);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t br = b0 + 32 * u;
              if (br >= no) break;
              const uint32_t orl = br + lane, pv = pvs[u], v = vs[u];
              const bool live = orl < no;
              const uint32_t last = min(br + 31, no - 1);
              uint32_t k;
              if (cur + 2 > nch || srel[cur + 2] > last) {
                k = cur + (cur + 1 < nch && srel[cur + 1] <= orl ? 1u : 0u);
              } else {
                uint32_t lo = cur, hi = nch;
                while (hi - lo > 1) {
                  const uint32_t mid = (lo + hi) >> 1;
                  if (srel[mid] <= orl) lo = mid; else hi = mid;
                }
                k = lo;
              }
              cur = __shfl_sync(0xffffffffu, k, 31);
              uint32_t prev = __shfl_up_sync(0xffffffffu, pv, 1);
              if (lane == 0) prev = static_cast<uint32_t>(carry);
              carry = __shfl_sync(0xffffffffu, pv, 31);
              const uint64_t idx = (ka + k) * a.chunk + pv;
              const bool pos_ok = pv < a.chunk && idx < n;
              const bool bad = live && (v >= exp_bins || !in_book(v) || !pos_ok ||
                                        (orl > srel[k] && prev >= pv));
              if (bad) {  // rare: the reference's checks in order (codec.py:446-536)
                const uint64_t o = o_lo + orl;
                if (v >= exp_bins) record_first(&a.status->first_inv[SZ_DEC_VALUE_DOMAIN], o);
                else if (!in_book(v)) record_first(&a.status->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
                if (pv >= a.chunk) record_first(&a.status->first_inv[SZ_DEC_POS_OVER_CHUNK], o);
                else if (idx >= n) record_first(&a.status->first_inv[SZ_DEC_POS_PAST_END], o);
                else if (orl > srel[k] && prev >= pv)
                  record_first(&a.status->first_inv[SZ_DEC_POS_NOT_INC], o);
              }
              const bool hit = live && pos_ok && idx >= s0 && idx < s1;
              const uint32_t hb = __ballot_sync(0xffffffffu, hit);
              if (!have_first && hb) {
                o_first = o_lo + br + (__ffs(hb) - 1);
                have_first = true;
              }
              const uint64_t o = o_lo + orl;
              if (hit && o >= o_first) stage(idx, o - o_first, v);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              pvs[u] = npvs[u];
              vs[u] = nvs[u];
            }
          }
        } else {
        uint64_t base = o_lo;
        for (; base + 32 * U <= o_hi; base += 32 * U) {
          uint64_t pvs[U];
          uint32_t vs[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            pvs[u] = load_pos<POSB>(a.positions, base + 32 * u + lane);
            vs[u] = a.values[base + 32 * u + lane];
          }
#pragma unroll
          for (int u = 0; u < U; ++u) one(base + 32 * u, pvs[u], vs[u]);
        }
        for (; base < o_hi; base += 32) {
          const uint64_t o = base + lane;
          one(base, o < o_hi ? load_pos<POSB>(a.positions, o) : 0,
              o < o_hi ? a.values[o] : 0u);
        }
        }
      }
      if (lane == 0) {
        S.ofirst[s] = o_first;
        S.vshift[s] = vshift;
      }
      __syncwarp();
      mbar_arrive(&S.staged[s]);
    }
    return;
  }

  // ------------------------------------------------------------ decode warps
  const bool check_range = p.n_entries < (1u << CB);
  for (uint32_t it = 0;; ++it) {
    const uint32_t s = it % kStages, ph = (it / kStages) & 1;
    mbar_wait(&S.full[s], ph);
    const uint64_t tile = S.meta[s];
    if (tile == ~0ull) break;
    const uint64_t tile_e0 = tile * TILE;
    const uint32_t full_slots = static_cast<uint32_t>(min(n - tile_e0, TILE) / EPV);
    const uint32_t cbytes = (full_slots * CBYTES) & ~15u;
    const uint32_t sbytes = (full_slots * SBYTES) & ~15u;
    mbar_wait(&S.staged[s], ph);
    const uint64_t ofirst = S.ofirst[s];
    const uint32_t vshift = S.vshift[s];
#pragma unroll
    for (int i = 0; i < kDecItems; ++i) {
      const uint32_t slot = i * kThreads + tid;
      const uint64_t e0 = tile_e0 + static_cast<uint64_t>(slot) * EPV;
      if (e0 >= n) continue;
      const int nv = e0 + EPV <= n ? EPV : static_cast<int>(n - e0);
      uint32_t cw[CWORDS], sw[SWORDS];
      if ((slot + 1) * CBYTES <= cbytes && (slot + 1) * SBYTES <= sbytes) {
        const uint8_t* cp = S.codes[s] + slot * CBYTES;
        const uint8_t* sp = S.sm[s] + slot * SBYTES;
        if constexpr (CBYTES == 16) {
          const uint4 v = *reinterpret_cast<const uint4*>(cp);
          cw[0] = v.x; cw[1] = v.y; cw[2] = v.z; cw[3] = v.w;
        } else if constexpr (CBYTES == 8) {
          const uint2 v = *reinterpret_cast<const uint2*>(cp);
          cw[0] = v.x; cw[1] = v.y;
        } else if constexpr (CBYTES == 12) {
          const uint32_t* q = reinterpret_cast<const uint32_t*>(cp);
          cw[0] = q[0]; cw[1] = q[1]; cw[2] = q[2];
        } else {
          const uint16_t* q = reinterpret_cast<const uint16_t*>(cp);
          cw[0] = q[0] | (static_cast<uint32_t>(q[1]) << 16);
          cw[1] = q[2];
        }
        if constexpr (SBYTES == 16) {
          const uint4 v = *reinterpret_cast<const uint4*>(sp);
          sw[0] = v.x; sw[1] = v.y; sw[2] = v.z; sw[3] = v.w;
        } else {
          const uint32_t* q = reinterpret_cast<const uint32_t*>(sp);
          sw[0] = q[0]; sw[1] = q[1]; sw[2] = q[2];
        }
      } else {
        ld_bytes_clipped<CBYTES>(a.codes, e0 * CB / 8, cw, a.codes_len);
        ld_bytes_clipped<SBYTES>(a.sm, e0 * SMB / 8, sw, a.sm_len);
      }
      if constexpr (kE5Fast) {
        // E5M2, 4-bit codes: placed-exponent pair tables + SWAR sign|mantissa
        uint32_t ow[8];
        uint32_t bad = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t w = cw[g >> 1];
          // u16 entries: the 64 commonest code pairs (both codes < 16, the
          // second < 4 — codes are frequency-ranked) sit in 32 distinct banks
          const uint32_t blo = (g & 1) ? ((w >> 15) & 0x1FEu) : ((w << 1) & 0x1FEu);
          const uint32_t bhi = (g & 1) ? ((w >> 23) & 0x1FEu) : ((w >> 7) & 0x1FEu);
          const uint32_t ex = __byte_perm(*reinterpret_cast<const uint16_t*>(e5tab + blo),
                                          *reinterpret_cast<const uint16_t*>(e5tab + bhi),
                                          0x5410);
          ow[g] = ex | e5m2_sm_bytes(group_bits<12>(sw, g));
        }
        if (check_range) {  // codebook < 16 entries: flag codes past its end
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t w = cw[g >> 1] >> (16 * (g & 1));
            const uint32_t l0 = lds_u32(lut2_base | ((w << 2) & 0x3FCu));
            const uint32_t l1 = lds_u32(lut2_base | ((w >> 6) & 0x3FCu));
            bad |= (((l0 >> 16) & 3) | (((l1 >> 16) & 3) << 2)) << (4 * g);
          }
        }
        if constexpr (SENT) bad &= ~S.bitmap[s][slot];  // marks are not dense codes
        if (bad) {
          if (nv < 32) bad &= (1u << nv) - 1u;
          if (bad) record_first(&a.status->first_inv[SZ_DEC_CODE_RANGE], e0 + (__ffs(bad) - 1));
        }
        uint32_t bm = S.bitmap[s][slot];
        const uint32_t bm0 = bm;
        if constexpr (kGroupMerge) {
          // group-wise PRMT merge of the placed exponent fields (bits 2-6),
          // branch-free: a group without escapes merges with the identity
          // selector (the slot's escape-free groups cost a few instructions
          // instead of a divergent branch per group)
          const uint32_t sf = S.slot_first[s][slot];
          const uint32_t first = bm ? sf : 0u;
          if (first + __popc(bm) <= static_cast<uint32_t>(kDecValCap<FMT>)) {
            const uint32_t vbase = smem_addr(S.vals[s]) + vshift;
            uint32_t r = first, nd_any = 0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const uint32_t mg = (bm >> (4 * g)) & 15u;
              uint32_t nd;
              const uint32_t t = merge_group(ow[g] >> 2 & 0x1F1F1F1Fu, mg, r, vbase, sel_base,
                                             d0 * 0x01010101u, &nd);
              ow[g] = (ow[g] & 0x83838383u) | ((t << 2) & 0x7C7C7C7Cu);
              nd_any |= nd;
              r += __popc(mg);
            }
            if (!SENT && nd_any)   // rare: the first escaped element with a non-dummy code
              first_nondummy<CB, CWORDS>(cw, bm, e0, a.status);
            bm = 0;
          }
        }
        while (bm) {  // rare: overwrite escaped exponent fields (bits 2-6 of the byte)
          const int j = __ffs(bm) - 1;
          bm &= bm - 1;
          const uint32_t code = (pick<CWORDS>(cw, j >> 3) >> (4 * (j & 7))) & 0xF;
          if (!SENT && code != 0) record_first(&a.status->first_inv[SZ_DEC_NONDUMMY], e0 + j);
          const uint32_t v = escape_value<kDecValCap<FMT>>(S.vals[s] + vshift, S.slot_first[s][slot], bm0,
                                                           j, ofirst, m, a.values);
          const int g = j >> 2, sh = 8 * (j & 3);
#pragma unroll
          for (int gg = 0; gg < G; ++gg)
            if (gg == g) ow[gg] = (ow[gg] & ~(0x7Cu << sh)) | (v << (sh + 2));
        }
        if (nv == EPV) st256(out_slot<WB>(a, e0), ow);
        else st_bytes_clipped<32>(a.out, e0 * WB, ow, n * WB);
        continue;
      }
      uint32_t eg[G], ag[G];
      uint32_t bad = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        uint32_t l0, l1;
        if constexpr (CB == 4) {
          // code bytes 2g, 2g+1 of the slot: word g/2, bit offset 16*(g&1)
          const uint32_t w = cw[g >> 1];
          if ((g & 1) == 0) {
            l0 = lds_u32(lut2_base | ((w << 2) & 0x3FCu));
            l1 = lds_u32(lut2_base | ((w >> 6) & 0x3FCu));
          } else {
            l0 = lds_u32(lut2_base | ((w >> 14) & 0x3FCu));
            l1 = lds_u32(lut2_base | ((w >> 22) & 0x3FCu));
          }
        } else {
          const uint32_t cb12 = group_bits<12>(cw, g);
          if (T12 && !check_range) {
            // the group's four exponents in one lookup (full 8-entry book)
            eg[g] = lds_u32(t12_base + (cb12 << 2));
            if constexpr (SMB == 8) ag[g] = sw[g];
            else if constexpr (SMB == 4) ag[g] = unpack_nib4(group_bits<16>(sw, g));
            else ag[g] = unpack_tri4(group_bits<12>(sw, g));
            continue;
          }
          l0 = lds_u32(lut2_base | ((cb12 << 2) & 0xFCu));
          l1 = lds_u32(lut2_base | ((cb12 >> 4) & 0xFCu));
        }
        eg[g] = __byte_perm(l0, l1, 0x5410);
        if (check_range) bad |= (((l0 >> 16) & 3) | (((l1 >> 16) & 3) << 2)) << (4 * g);
        if constexpr (SMB == 8) ag[g] = sw[g];
        else if constexpr (SMB == 4) ag[g] = unpack_nib4(group_bits<16>(sw, g));
        else ag[g] = unpack_tri4(group_bits<12>(sw, g));
      }
      if constexpr (SENT) {  // marks are not dense codes
        if constexpr (EPV == 32) bad &= ~S.bitmap[s][slot];
        else bad &= ~((S.bitmap[s][slot >> 1] >> (16 * (slot & 1))) & 0xFFFFu);
      }
      if (bad) {
        if (nv < 32) bad &= (1u << nv) - 1u;
        if (bad) record_first(&a.status->first_inv[SZ_DEC_CODE_RANGE], e0 + (__ffs(bad) - 1));
      }
      uint32_t bm;
      if constexpr (EPV == 32) bm = S.bitmap[s][slot];
      else bm = (S.bitmap[s][slot >> 1] >> (16 * (slot & 1))) & 0xFFFFu;
      const uint32_t bm0 = bm;
      if constexpr (kGroupMerge) {
        // escaped exponents merged group by group (merge_group): no loop
        // over the escapes, so escape-dense slots do not serialise the warp;
        // branch-free (escape-free groups merge with the identity selector)
        const uint32_t sf = S.slot_first[s][slot];
        const uint32_t first = bm ? sf : 0u;
        if (first + __popc(bm) <= static_cast<uint32_t>(kDecValCap<FMT>)) {
          const uint32_t vbase = smem_addr(S.vals[s]) + vshift;
          uint32_t r = first, nd_any = 0;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t mg = (bm >> (4 * g)) & 15u;
            uint32_t nd;
            eg[g] = merge_group(eg[g], mg, r, vbase, sel_base, d0 * 0x01010101u, &nd);
            nd_any |= nd;
            r += __popc(mg);
          }
          if (!SENT && nd_any)   // rare: the first escaped element with a non-dummy code
            first_nondummy<CB, CWORDS>(cw, bm, e0, a.status);
          bm = 0;
        }
      }
      // beyond the staged values (tiles with more escapes than kDecValCap):
      // the compact loop over set bits, values from global memory (the
      // register arrays are indexed through selects, never dynamically)
      while (bm) {
        const int j = __ffs(bm) - 1;
        bm &= bm - 1;
        uint32_t code;
        if constexpr (CB == 4) {
          code = (pick<CWORDS>(cw, j >> 3) >> (4 * (j & 7))) & 0xF;
        } else {
          const int bit = 3 * j;
          const uint64_t lo = pick<CWORDS>(cw, bit >> 5);
          const uint64_t hi = pick<CWORDS>(cw, (bit >> 5) + 1);
          code = static_cast<uint32_t>(((hi << 32) | lo) >> (bit & 31)) & 7;
        }
        if (!SENT && code != 0) record_first(&a.status->first_inv[SZ_DEC_NONDUMMY], e0 + j);
        const uint32_t v = escape_value<kDecValCap<FMT>>(S.vals[s] + vshift, S.slot_first[s][slot], bm0,
                                                         j, ofirst, m, a.values);
        const int g = j >> 2, sh = 8 * (j & 3);
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          if (gg == g) eg[gg] = (eg[gg] & ~(0xFFu << sh)) | (v << sh);
      }
      uint32_t ow[8];
#pragma unroll
      for (int g = 0; g < G; ++g) rebuild_group<FMT>(eg[g], ag[g], ow, g);
      if (nv == EPV) st256(out_slot<WB>(a, e0), ow);
      else st_bytes_clipped<32>(a.out, e0 * WB, ow, n * WB);
    }
    mbar_arrive(&S.empty[s]);
  }
}

__global__ void check_values_kernel(const uint8_t* __restrict__ values, uint64_t m,
                                    const __grid_constant__ sz_params p, sz_decode_status* st) {
  const uint32_t exp_bins = 1u << (p.fmt == SZ_BF16 ? 8 : (p.fmt == SZ_E5M2 ? 5 : 4));
  for (uint64_t o = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; o < m;
       o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = values[o];
    if (v >= exp_bins) record_first(&st->first_inv[SZ_DEC_VALUE_DOMAIN], o);
    else if (!(p.enc_lut[v] & 0x10)) record_first(&st->first_inv[SZ_DEC_VALUE_IN_BOOK], o);
  }
}

}  // namespace sz

// ============================================================ host dispatch
namespace {
using namespace sz;

constexpr int kDecodeItems = 2;

uint64_t decode_tile_for(uint32_t fmt) {
  return static_cast<uint64_t>(kDecodeItems) * kThreads * (fmt == SZ_BF16 ? 16 : 32);
}

struct DecodeWs {
  uint64_t* offsets;
  uint64_t* off_states;
  unsigned long long* off_counter;
  uint64_t* dec_states;
  unsigned long long* dec_counter;
  uint64_t* t_states;    // marked (K3e): look-back states of the tile-count scan
  unsigned long long* t_counter;
  uint64_t* tile_offsets;  // marked (K3e): first ordinal of every decode tile
  uint32_t* tile_marks;  // sentinel / marked: escapes per decode tile
  uint32_t* mark_bits;   // sentinel / marked: one bit per element, read by the stagers
  size_t zero_bytes;  // prefix of the workspace that must be zeroed
  size_t total;
};

// Escape-dense chunk-relative streams take the K3e path (bitmap pre-pass)
// when the declared M reaches 1/kDenseDiv of N.  The crossover was measured
// with SZ_DEC_MARKED=0/1 (forces either path; tuning and tests only) at 2^31
// words (profiles/bench_dense_r02.jsonl): with the branch-free group merge
// the stager walk wins below ~1.8% escapes, K3e above ~2% (BF16 7.89%:
// 1227 -> 1921 GB/s).
constexpr uint64_t kDenseDiv = 50;
int marked_override() {
  const char* e = getenv("SZ_DEC_MARKED");   // read per call: tests force both paths
  return e && *e ? atoi(e) : -1;
}
bool want_marked(uint64_t n, uint64_t m, const sz_params* p) {
  if (p->sentinel || p->abs32 || p->chunk_size < kMarkMinChunk || m == 0) return false;
  const int o = marked_override();
  if (o >= 0) return o != 0;
  return m * kDenseDiv >= n;
}

DecodeWs carve(void* base, uint64_t n, const sz_params* p, bool marked) {
  DecodeWs w{};
  const bool chunked = !p->sentinel && !p->abs32;
  const uint64_t tile = decode_tile_for(p->fmt);
  const uint64_t dtiles = (n + tile - 1) / tile;
  // scanned counts: per-chunk escape counts, or (sentinel) per-tile marks
  // abs32: the scanned array is replaced by per-tile ordinal bounds (K3a)
  const uint64_t nchunks = chunked ? (n + p->chunk_size - 1) / p->chunk_size
                                   : (p->sentinel ? dtiles : 0);
  const uint64_t nbounds = p->abs32 ? dtiles + 1 : 0;
  const uint64_t otiles = nchunks ? offsets_tiles(nchunks) : 0;
  const uint64_t ttiles = marked ? offsets_tiles(dtiles) : 0;
  // layout in u64 units from the (256-aligned) base; zeroed region first:
  // look-back states + counters (+ abs32 bounds)
  uint64_t at = 0;
  const uint64_t i_off_states = at; at += otiles;
  const uint64_t i_off_counter = at; at += 1;
  const uint64_t i_dec_states = at; at += dtiles;
  const uint64_t i_dec_counter = at; at += 1;
  const uint64_t i_t_states = at; at += ttiles;
  const uint64_t i_t_counter = at; at += marked ? 1 : 0;
  // offsets start 16-byte aligned (the scan's vector stores)
  at = (at + 1) & ~1ull;
  const uint64_t i_offsets = at;
  at += nbounds;
  w.zero_bytes = at * sizeof(uint64_t);
  at = i_offsets + (nchunks ? nchunks + 1 : nbounds);
  at = (at + 1) & ~1ull;
  const uint64_t i_tile_offsets = at; at += marked ? dtiles + 1 : 0;
  const bool marks = p->sentinel || marked;
  const uint64_t tm_bytes = marks ? dtiles * sizeof(uint32_t) : 0;
  const uint64_t b_tile_marks = at * sizeof(uint64_t);
  // (16-byte aligned: the stagers read it with vector loads)
  const uint64_t b_mark_bits = (b_tile_marks + tm_bytes + 15) & ~15ull;
  const uint64_t nbits_words = marks ? dtiles * (tile / 32) : 0;
  w.total = b_mark_bits + nbits_words * sizeof(uint32_t) + 256;
  uint8_t* b8 = static_cast<uint8_t*>(base);
  uint64_t* b = static_cast<uint64_t*>(base);
  w.off_states = b + i_off_states;
  w.off_counter = reinterpret_cast<unsigned long long*>(b + i_off_counter);
  w.dec_states = b + i_dec_states;
  w.dec_counter = reinterpret_cast<unsigned long long*>(b + i_dec_counter);
  w.t_states = b + i_t_states;
  w.t_counter = reinterpret_cast<unsigned long long*>(b + i_t_counter);
  w.offsets = b + i_offsets;
  w.tile_offsets = b + i_tile_offsets;
  w.tile_marks = reinterpret_cast<uint32_t*>(b8 + b_tile_marks);
  w.mark_bits = reinterpret_cast<uint32_t*>(b8 + b_mark_bits);
  return w;
}

// Exclusive scan of n u32 counts into u64 offsets (K3's kernels): decoupled
// look-back up to 32 CTAs, reduce-then-scan beyond.
cudaError_t launch_scan(OffsetsArgs oa, cudaStream_t s) {
  oa.num_tiles = offsets_tiles(oa.n_counts);
  cudaError_t e = cudaSuccess;
  if (oa.num_tiles > 32) {
    // many CTAs: per-CTA sums in the look-back state array (unused then)
    e = launch_pdl(offsets_sums_kernel, dim3(static_cast<unsigned>(oa.num_tiles)),
                   dim3(kThreads), 0, s, oa, oa.states);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    oa.sums = oa.states;
  }
  e = launch_pdl(offsets_kernel, dim3(static_cast<unsigned>(oa.num_tiles)), dim3(kThreads), 0,
                 s, oa);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

template <int POSB>
cudaError_t launch_marks(const MarkArgs& ma, cudaStream_t s) {
  auto kern = escape_marks_kernel<POSB>;
  const int smem = static_cast<int>(sizeof(MarkSmem)) * kMarkWarps;
  const KernelSetup ks = kernel_setup(reinterpret_cast<const void*>(kern), smem, kMarkWarps * 32);
  if (ks.err != cudaSuccess) return ks.err;
  const uint64_t want = static_cast<uint64_t>(ks.sms) * (ks.per_sm < 1 ? 1 : ks.per_sm);
  const uint64_t ctas = (ma.n_windows + kMarkWarps - 1) / kMarkWarps;
  const unsigned grid = static_cast<unsigned>(ctas < want ? ctas : want);
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kMarkWarps * 32), smem, s, ma);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

// Explicit modes: persistent warp-specialised kernel.
template <int FMT, int CB, int POSB>
cudaError_t launch_persistent(const sz_params& p, const DecodeArgs& a, cudaStream_t s) {
  auto kern = decode_persistent<FMT, CB, POSB>;
  const int smem = static_cast<int>(sizeof(DecSmem<FMT, kDecStages<FMT, CB, POSB>, CB>));
  const KernelSetup ks = kernel_setup(reinterpret_cast<const void*>(kern), smem, kDecThreads);
  if (ks.err != cudaSuccess) return ks.err;
  const int per_sm = ks.per_sm < 1 ? 1 : ks.per_sm;
  const uint64_t want = static_cast<uint64_t>(ks.sms) * per_sm;
  const unsigned grid = static_cast<unsigned>(a.num_tiles < want ? a.num_tiles : want);
  cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kDecThreads), smem, s, p, a);
  return e == cudaSuccess ? cudaGetLastError() : e;
}
template <int FMT, int CB>
cudaError_t dec_pos(int posb, const sz_params& p, const DecodeArgs& a, cudaStream_t s) {
  switch (posb) {
    case 0: return launch_persistent<FMT, CB, 0>(p, a, s);
    case 1: return launch_persistent<FMT, CB, 1>(p, a, s);
    case 2: return launch_persistent<FMT, CB, 2>(p, a, s);
    case kPosMarked: return launch_persistent<FMT, CB, kPosMarked>(p, a, s);
    default: return launch_persistent<FMT, CB, 4>(p, a, s);
  }
}
template <int FMT>
cudaError_t dec_cb(int posb, const sz_params& p, const DecodeArgs& a, cudaStream_t s) {
  return p.code_bits == 4 ? dec_pos<FMT, 4>(posb, p, a, s) : dec_pos<FMT, 3>(posb, p, a, s);
}

}  // namespace

extern "C" {

int sz_record_cuda(cudaError_t e);
int sz_check_params(const sz_params* p, int decode_side);

size_t sz_decode_workspace_bytes(uint64_t n, uint64_t m, const sz_params* p) {
  if (!p || p->fmt > SZ_E4M3 || p->chunk_size == 0) return 0;
  return carve(nullptr, n, p, want_marked(n, m, p)).total;
}

}  // extern "C"

namespace {
// Shared body of sz_decode (contiguous output) and sz_decode_segments (paged
// output: d_words_out null, segment table + log2 segment bytes).
int decode_impl(const sz_encoded_in* in, const sz_params* p, void* d_words_out,
                const uint64_t* seg_addrs, uint32_t seg_shift, sz_decode_status* d_status,
                void* d_ws, size_t ws_bytes, void* stream) {
  if (int rc = sz_check_params(p, 1)) return rc;
  if (!in || (!d_words_out && !seg_addrs) || !d_status || in->n_elements == 0)
    return SZ_ECONFIG;
  if (!in->d_n_escapes && in->n_escapes > in->n_elements) return SZ_ECONFIG;
  // device-resident M: n_escapes is the escape buffers' capacity (0 = N);
  // every kernel reads min(*d_n_escapes, m)
  const uint64_t n = in->n_elements;
  const uint64_t m = in->d_n_escapes ? (in->n_escapes ? min(in->n_escapes, n) : n)
                                     : in->n_escapes;
  if ((reinterpret_cast<uintptr_t>(d_words_out) & 31) ||
      (reinterpret_cast<uintptr_t>(in->d_codes) & 15) || (reinterpret_cast<uintptr_t>(in->d_sm) & 15))
    return SZ_EALIGN;
  // the escape-dense path when the workspace was sized for it (a caller may
  // size it with another M than the one declared here)
  const bool marked = want_marked(n, m, p) && ws_bytes >= carve(nullptr, n, p, true).total;
  if (ws_bytes < carve(nullptr, n, p, marked).total) return SZ_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool chunked = !p->sentinel && !p->abs32;
  const int sm_bits = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 3 : 4);
  DecodeWs w = carve(d_ws, n, p, marked);
  const uint64_t nchunks = chunked ? (n + p->chunk_size - 1) / p->chunk_size : 0;
  if (chunked && in->n_counts != nchunks) return SZ_ECONFIG;  // host raises first
  if (!in->d_n_escapes && m && (!in->d_values || (!p->sentinel && !in->d_positions)))
    return SZ_ECONFIG;

  cudaError_t e = cudaMemsetAsync(d_status, 0, sizeof(sz_decode_status), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_ws, 0, w.zero_bytes, s);
  if (e != cudaSuccess) return sz_record_cuda(e);

  const uint64_t dtiles = (n + decode_tile_for(p->fmt) - 1) / decode_tile_for(p->fmt);
  if (p->sentinel) {
    // K3s: marks per decode tile, then their scan (tile ordinal bases) below
    const uint64_t want = (dtiles + kWarps - 1) / kWarps;  // one warp per tile
    const unsigned g = static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
    const uint64_t clen = (n * p->code_bits + 7) / 8;
    const uint32_t slots = kDecSlots;
    const uint8_t* codes = static_cast<const uint8_t*>(in->d_codes);
    switch (p->fmt * 2 + (p->code_bits == 4)) {
      case 0: marks_kernel<SZ_BF16, 3><<<g, kThreads, 0, s>>>(codes, n, clen, dtiles, slots, w.tile_marks, w.mark_bits); break;
      case 1: marks_kernel<SZ_BF16, 4><<<g, kThreads, 0, s>>>(codes, n, clen, dtiles, slots, w.tile_marks, w.mark_bits); break;
      case 2: marks_kernel<SZ_E5M2, 3><<<g, kThreads, 0, s>>>(codes, n, clen, dtiles, slots, w.tile_marks, w.mark_bits); break;
      case 3: marks_kernel<SZ_E5M2, 4><<<g, kThreads, 0, s>>>(codes, n, clen, dtiles, slots, w.tile_marks, w.mark_bits); break;
      case 4: marks_kernel<SZ_E4M3, 3><<<g, kThreads, 0, s>>>(codes, n, clen, dtiles, slots, w.tile_marks, w.mark_bits); break;
      default: marks_kernel<SZ_E4M3, 4><<<g, kThreads, 0, s>>>(codes, n, clen, dtiles, slots, w.tile_marks, w.mark_bits); break;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return sz_record_cuda(e);
  }
  if (p->abs32) {
    const unsigned g = static_cast<unsigned>(device_sms() * 8);
    abs_bounds_kernel<<<g, kThreads, 0, s>>>(static_cast<const uint32_t*>(in->d_positions),
                                             in->d_n_escapes, m, n, decode_tile_for(p->fmt),
                                             dtiles, w.offsets);
    e = cudaGetLastError();
    if (e != cudaSuccess) return sz_record_cuda(e);
  }
  if (chunked || p->sentinel) {
    OffsetsArgs oa{};
    oa.m_ptr = in->d_n_escapes;
    oa.counts = p->sentinel ? w.tile_marks : in->d_counts;
    oa.sentinel = p->sentinel ? 1 : 0;
    oa.n_counts = p->sentinel ? dtiles : nchunks;
    oa.m = m;
    oa.offsets = w.offsets;
    oa.states = w.off_states;
    oa.tile_counter = w.off_counter;
    oa.status = d_status;
    e = launch_scan(oa, s);
    if (e != cudaSuccess) return sz_record_cuda(e);
  }
  if (marked) {
    // K3e: escape bitmap + per-tile counts + every per-ordinal check, then
    // the tile counts' scan (first ordinal of every decode tile)
    MarkArgs ma{};
    ma.m_ptr = in->d_n_escapes;
    ma.m = m;
    ma.offsets = w.offsets;
    ma.positions = in->d_positions;
    ma.values = in->d_values;
    ma.n = n;
    ma.n_windows = (n + kMarkWin - 1) / kMarkWin;
    ma.chunk = p->chunk_size;
    ma.tile_words = static_cast<uint32_t>(decode_tile_for(p->fmt) / 32);
    ma.n_words = dtiles * ma.tile_words;
    ma.exp_bins = 1u << (p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 5 : 4));
    // valid escape values: inside the exponent domain and outside the book
    for (uint32_t i = 0; i < ma.exp_bins && i < 256; ++i)
      ma.esc_ok[i >> 5] |= ((p->enc_lut[i] >> 4) & 1u) << (i & 31);
    ma.mark_bits = w.mark_bits;
    ma.tile_marks = w.tile_marks;
    ma.status = d_status;
    e = p->chunk_size <= 256 ? launch_marks<1>(ma, s) : launch_marks<2>(ma, s);
    if (e != cudaSuccess) return sz_record_cuda(e);
    OffsetsArgs ta{};
    ta.counts = w.tile_marks;
    ta.n_counts = dtiles;
    ta.offsets = w.tile_offsets;
    ta.states = w.t_states;
    ta.tile_counter = w.t_counter;
    e = launch_scan(ta, s);
    if (e != cudaSuccess) return sz_record_cuda(e);
  }

  DecodeArgs a{};
  a.m_ptr = in->d_n_escapes;
  a.codes = static_cast<const uint8_t*>(in->d_codes);
  a.sm = static_cast<const uint8_t*>(in->d_sm);
  a.offsets = marked ? w.tile_offsets : w.offsets;
  a.positions = in->d_positions;
  a.values = in->d_values;
  a.n = n;
  a.m = m;
  a.out = static_cast<uint8_t*>(d_words_out);
  a.seg_addrs = seg_addrs;
  a.seg_shift = seg_shift;
  a.status = d_status;
  a.states = w.dec_states;
  a.tile_counter = w.dec_counter;
  a.mark_bits = w.mark_bits;
  a.num_tiles = (n + decode_tile_for(p->fmt) - 1) / decode_tile_for(p->fmt);
  a.n_chunks = nchunks;
  a.codes_len = (n * p->code_bits + 7) / 8;
  a.sm_len = (n * sm_bits + 7) / 8;
  a.chunk = p->chunk_size;
  a.chunk_shift = (p->chunk_size & (p->chunk_size - 1)) == 0 ? __builtin_ctz(p->chunk_size) : -1;
  const int posb = p->sentinel ? 0
                 : p->abs32  ? 4
                 : marked    ? kPosMarked
                             : (p->chunk_size <= 256 ? 1 : 2);
  switch (p->fmt) {
    case SZ_BF16: e = dec_cb<SZ_BF16>(posb, *p, a, s); break;
    case SZ_E5M2: e = dec_cb<SZ_E5M2>(posb, *p, a, s); break;
    default: e = dec_cb<SZ_E4M3>(posb, *p, a, s); break;
  }
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}
}  // namespace

extern "C" {

int sz_decode(const sz_encoded_in* in, const sz_params* p, void* d_words_out,
              sz_decode_status* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_words_out) return SZ_ECONFIG;
  return decode_impl(in, p, d_words_out, nullptr, 0, d_status, d_ws, ws_bytes, stream);
}

int sz_decode_segments(const sz_encoded_in* in, const sz_params* p, const uint64_t* d_seg_addrs,
                       uint64_t n_segs, uint64_t seg_bytes, sz_decode_status* d_status,
                       void* d_ws, size_t ws_bytes, void* stream) {
  if (!p || !in || !d_seg_addrs || n_segs == 0 || seg_bytes < 32 ||
      (seg_bytes & (seg_bytes - 1)))
    return SZ_ECONFIG;
  const uint64_t wb = p->fmt == SZ_BF16 ? 2 : 1;
  if (in->n_elements != n_segs * seg_bytes / wb) return SZ_ECONFIG;
  return decode_impl(in, p, nullptr, d_seg_addrs, static_cast<uint32_t>(__builtin_ctzll(seg_bytes)),
                     d_status, d_ws, ws_bytes, stream);
}

int sz_check_values(const uint8_t* d_values, uint64_t m, const sz_params* p,
                    sz_decode_status* d_status, void* stream) {
  if (int rc = sz_check_params(p, 1)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_status, 0, sizeof(sz_decode_status), s);
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (!m) return SZ_OK;
  uint64_t g = (m + kThreads - 1) / kThreads;
  if (g > 148 * 8) g = 148 * 8;
  check_values_kernel<<<static_cast<unsigned>(g), kThreads, 0, s>>>(d_values, m, *p, d_status);
  e = cudaGetLastError();
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

}  // extern "C"
