// sz_encode.cu — K2: SplitZip encoder for sm_100a.
//
// Replaces codec.py:299-321 (encode) and its byte-identical Quad64 variant
// codec.py:324-401 (encode_quad).  Three kernels on one stream:
//
// K2a  encode_tiles — persistent, warp-specialised, one CTA per SM (20 warps):
//   warp 16    PRODUCER claims 32 KiB tiles of input words (global counter)
//                       and streams them into a 4-deep shared-memory ring by
//                       TMA: a 128B-swizzled 2-D tensor-map box per full tile
//                       (contiguous input, or paged input inside a known VA
//                       window), else 1-D bulk copies; completion counted on
//                       an mbarrier.
//   warps 0-15 DENSE    per 32-byte slot (16 BF16 / 32 FP8 words): four
//                       lane-table lookups per 4-element group
//                       (t4[k][e] = code << CB*k | escape << 16+k, from the
//                       marked LUT of encode_quad, codec.py:340-342) give the
//                       packed 4-bit / 3-bit code group and its escape flags;
//                       the sign|mantissa plane is gathered with permutes and
//                       multiplies; both planes are vector-stored.  The slot's
//                       escape bitmask and compact (element, raw exponent)
//                       records stay in shared memory.
//   warps 17-19 WRITER  per tile: popc of the slot masks + warp scan = the
//                       tile-local escape order, per-chunk counts
//                       (codec.py:292-295), escape records written in
//                       ascending element order into the tile's scratch slot.
//   No CTA ever waits for another, so the stream runs at HBM speed.
// K2b  escape_gather — decoupled look-back prefix over the per-tile escape
//   counts, then coalesced moves of every regular tile's records to their
//   global ordinals in escape_positions / escape_values (codec.py:281-296);
//   tiles whose escapes overflowed the scratch slot are listed for K2c.
// K2c  escape_heavy — one CTA per listed tile re-derives its escapes from the
//   input in element order.
#include <cstdio>
#include <cstdlib>

#include <cuda.h>           // CUtensorMap (types only; the encoder entry point
#include <cudaTypedefs.h>   // comes from cudaGetDriverEntryPoint — no -lcuda)

#include <type_traits>

#include "sz_common.cuh"
#include "sz_scan.cuh"

namespace sz {

constexpr int kEncDenseWarps = 16;
constexpr int kEncDense = kEncDenseWarps * 32;          // 512 dense threads
constexpr int kEncItems = 2;                            // slots per dense thread
constexpr int kEncSlots = kEncItems * kEncDense;         // 1024 slots per tile
constexpr int kEncTileBytes = kEncSlots * 32;           // 32 KiB of input words
constexpr int kEncInStages = 4;
constexpr int kEncScanSlots = 8;
// Escape records per tile the dense warps can stage in shared memory (12.5%
// of a BF16 tile, 6.25% of an FP8 tile); a tile past it is re-derived by K2c.
// BF16 (7 writer warps) 1984; FP8 (3 writer warps, twice the elements per
// tile) 2400 — what the shared memory left by the rest of EncSmem holds.
#ifndef SZ_FP8_ESC_CAP
#define SZ_FP8_ESC_CAP 2400
#endif
template <int FMT>
constexpr int kEscValCap = FMT == SZ_BF16 ? 1984 : SZ_FP8_ESC_CAP;
// Scratch records per tile in global memory: 1/8 of the tile's elements
// (2048 BF16 / 4096 FP8 — a top-8 3-bit book's ~7% escapes fit), so the
// scratch is n/8 records; tiles with more escapes go to K2c.
template <int FMT>
constexpr uint32_t kTileCap = kEncSlots * kEpv<FMT> / 8 < kEscValCap<FMT>
                                  ? kEncSlots * kEpv<FMT> / 8 : kEscValCap<FMT>;
// Writer warps: the escape records' placement is a per-tile serial chain
// per writer, so escape-dense BF16 tiles want many (7: 16 + 1 + 7 = 24 warps
// at 80 registers); the FP8 dense warps of realistic books are issue-bound
// and need the registers (3: 20 warps at 96).  E5M2 with 3-bit codes (top-8
// books: ~7% escapes, twice BF16's per tile) was writer-bound with 3 (per-role
// cycle counters: writers busy 95% of the kernel, the producer waiting on
// their scan slots): 7 writers at 80 registers, 7 scan slots so the shared
// memory fits — 1045 -> 1183 GB/s; E4M3 3-bit books are sparse and lost 5%
// with 7, so they keep 3.  Warp counts stay multiples of 4 so the register
// file splits evenly.
template <int FMT, int CB>
constexpr int kWriterWarps = FMT == SZ_BF16 ? 7 : (FMT == SZ_E5M2 && CB == 3 ? 7 : 3);
template <int FMT, int CB>
constexpr int kScanSlots = FMT == SZ_E5M2 && CB == 3 ? 7 : kEncScanSlots;
template <int FMT, int CB>
constexpr int kEncThreads = kEncDense + 32 * (1 + kWriterWarps<FMT, CB>);
constexpr int kProducerWarp = kEncDenseWarps;           // warp 16
constexpr int kWriterWarp0 = kEncDenseWarps + 1;        // warps 17..

struct EncodeArgs {
  const uint8_t* words;
  uint64_t n;
  uint8_t* codes;
  uint8_t* sm;
  uint32_t* counts;
  uint64_t num_tiles;
  uint64_t n_chunks;
  uint64_t codes_len;
  uint64_t sm_len;
  uint32_t chunk;
  int32_t chunk_shift;   // log2(chunk) when a power of two, else -1
  int32_t counts_mode;   // 0 none, 1 direct from the scan, 2 atomics (pre-zeroed)
  unsigned long long* tile_counter;
  uint32_t* tile_esc;    // per-tile escape count
  uint8_t* scr_pos;      // kTileCap positions per tile (POSB bytes each)
  uint8_t* scr_val;      // kTileCap raw exponents per tile
  const uint64_t* escape_base;  // append mode: global ordinal offset (or null)
  uint64_t* base_snapshot;      // workspace copy of *escape_base for K2b
  unsigned long long* dbg;  // optional per-role cycle counters (SZ_DEBUG_TIMERS)
  uint32_t lut_stride;      // 4 (byte stride of the T4 tables; see t4_group)
  uint32_t one;             // 1 (sum4)
  int32_t use_tmap;         // full tiles arrive by 2-D tensor TMA, 128B-swizzled
  // Segmented (paged) input: when non-null the logical
  // stream is segment i (2^seg_shift bytes) at seg_addrs[i], i = 0, 1, ...
  const uint64_t* seg_addrs;
  uint32_t seg_shift;
  uint32_t k_lo, k_hi;      // 1057 << 10, 1057 (e5m2_sm_hi)
  // segmented input with a tensor map over the virtual-address window that
  // holds every segment: full tiles arrive as 2-D boxes of min(segment,
  // tile) bytes at row (addr - seg_va_lo) / 128, 128B-swizzled like the
  // contiguous path (use_tmap is then set too)
  uint64_t seg_va_lo;
  int32_t seg_tmap;
};

template <int FMT, int CB>
struct EncSmem {
  static constexpr int Q = kScanSlots<FMT, CB>;
  // 1024-aligned: the 128B-swizzle pattern of tensor TMA is a function of
  // shared-address bits 7-9
  alignas(1024) uint8_t in[kEncInStages][kEncTileBytes];
  uint32_t fmask[Q][kEncSlots];  // at fsw(slot)
  // the tile's escape records, (tile-local element index, raw exponent), in
  // arbitrary order (one shared atomic per slot with escapes); the writer
  // derives each one's rank from fmask
  uint16_t esc_idx[Q][kEscValCap<FMT>];
  uint8_t esc_val[Q][kEscValCap<FMT>];
  uint32_t esc_n[Q];
  uint16_t slot_pref[kWriterWarps<FMT, CB>][kEncSlots];  // per-slot exclusive escape prefix, at fsw(slot)
  uint64_t meta[Q];      // tile id (~0 = end of work)
  uint64_t full[kEncInStages];       // producer -> dense (TMA bytes)
  uint64_t in_empty[kEncInStages];   // dense -> producer
  uint64_t computed[Q];  // dense -> writer
  uint64_t scan_empty[Q];// writer -> producer
};

// Shared-memory index of a slot's escape mask (and slot prefix).  Dense warps
// write 32 consecutive slots per warp; writer lane L reads its own 32
// consecutive slots L*32 + j, which in a linear layout all sit in one bank
// (32-way conflicts).  XOR-ing bits 5-9 of the slot into bits 0-4
// (bits 5-7 -> 2-4, bits 8-9 -> 0-1) makes both patterns conflict-free, and
// keeps every aligned group of 4 slots together (permuted inside), so 16-byte
// reads of 4 masks stay conflict-free across each 8-lane phase too.
__device__ __forceinline__ uint32_t fsw_key(uint32_t row) {  // row = slot >> 5
  return ((row & 7u) << 2) | ((row >> 3) & 3u);
}
__device__ __forceinline__ uint32_t fsw(uint32_t slot) { return slot ^ fsw_key(slot >> 5); }

// ---------------------------------------------------------------- T4 tables
// Lane tables for 4-bit codes (the north-star configuration):
//   t4[k][e] = code(e) << 4k  |  escape(e) << (16 + k)
// so the OR of the four lane-k lookups of a 4-element group is that group's
// packed nibble group (bits 0-15, element 0 in the low nibble — the order of
// formats.py:180-183) with its escape flags in bits 16-19.  One lookup per
// element replaces lookup + byte merge + nibble pack + flag extraction.
// E5M2: 32 entries per lane, lanes 128 B apart; the entry address is the
// exponent field itself (x & 0x7C = 4e) spliced into the table base by one
// PRMT.  BF16: 256 entries per lane, lanes 1 KB apart; 4e = (x >> 5) & 0x3FC.
// E5M2 alternative (-DSZ_E5_FULL_BYTE, off): lanes indexed by the whole byte,
// 256 entries each, every entry also carrying the element's 3-bit
// sign|mantissa symbol at bit 20 + 3k, so the OR of a group's four lookups is
// codes | flags | SM group — 37% fewer ALU instructions, but the byte index
// spreads a warp's lookups over ~2.4 distinct words per bank (sign and
// mantissa bits are uniform), and the shared-memory pipe becomes the limit:
// measured 2076 vs 2514 GB/s on B200.  The default indexes by exponent only
// (16 hot entries per lane table: conflict-free).
#ifdef SZ_E5_FULL_BYTE
constexpr bool kE5FullByte = true;
#else
constexpr bool kE5FullByte = false;
#endif
template <int FMT>
constexpr int kT4Entries = (FMT == SZ_BF16 || (FMT == SZ_E5M2 && kE5FullByte)) ? 256
                           : (FMT == SZ_E5M2 ? 32 : 16);
// Lane tables for every code width: with 3-bit codes the four lookups of a
// group sum to its 12-bit code group (bits 0-11), flags still in bits 16-19.

template <int OFF>
__device__ __forceinline__ uint32_t lds_u32_off(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(saddr), "n"(OFF));
  return v;
}

// Codes + flags of group g (elements 4g..4g+3) of a 32-byte slot.
__device__ __forceinline__ uint32_t w_mad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Sum of four lookups whose bits are disjoint (== their OR) as three IMADs
// with the opaque kernel argument 1: the FMA pipe adds, the ALU pipe is free.
__device__ __forceinline__ uint32_t sum4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                         uint32_t one) {
  return w_mad(w_mad(t0, one, t1), one, w_mad(t2, one, t3));
}

template <int FMT>
__device__ __forceinline__ uint32_t t4_group(const uint32_t (&x)[8], int g, uint32_t base,
                                             uint32_t stride, uint32_t one) {
  if constexpr (FMT == SZ_E5M2 && kE5FullByte) {
    // entry address = base + 4 * byte as ONE IMAD: `stride` is the kernel
    // argument 4, opaque to ptxas, so it cannot strength-reduce the multiply
    // into an ALU-pipe LEA/shift — the FMA pipe is otherwise idle here.
    const uint32_t w = x[g];
    const uint32_t t0 = lds_u32_off<0>(w_mad(w & 0xFFu, stride, base));
    const uint32_t t1 = lds_u32_off<1024>(w_mad(__byte_perm(w, 0, 0x4441), stride, base));
    const uint32_t t2 = lds_u32_off<2048>(w_mad(__byte_perm(w, 0, 0x4442), stride, base));
    const uint32_t t3 = lds_u32_off<3072>(w_mad(w >> 24, stride, base));
    return t0 | t1 | t2 | t3;
  } else if constexpr (FMT == SZ_E5M2) {
    const uint32_t f = x[g] & 0x7C7C7C7Cu;  // byte k = 4 * exponent of element k
    const uint32_t t0 = lds_u32_off<0>(__byte_perm(f, base, 0x7650));
    const uint32_t t1 = lds_u32_off<128>(__byte_perm(f, base, 0x7651));
    const uint32_t t2 = lds_u32_off<256>(__byte_perm(f, base, 0x7652));
    const uint32_t t3 = lds_u32_off<384>(__byte_perm(f, base, 0x7653));
    return sum4(t0, t1, t2, t3, one);
  } else if constexpr (FMT == SZ_E4M3) {
    const uint32_t f = (x[g] >> 1) & 0x3C3C3C3Cu;  // byte k = 4 * exponent (4 bits)
    const uint32_t t0 = lds_u32_off<0>(__byte_perm(f, base, 0x7650));
    const uint32_t t1 = lds_u32_off<64>(__byte_perm(f, base, 0x7651));
    const uint32_t t2 = lds_u32_off<128>(__byte_perm(f, base, 0x7652));
    const uint32_t t3 = lds_u32_off<192>(__byte_perm(f, base, 0x7653));
    return sum4(t0, t1, t2, t3, one);
  } else {
    const uint32_t f0 = (x[2 * g] >> 5) & 0x03FC03FCu;      // 4e of elements 4g, 4g+1
    const uint32_t f1 = (x[2 * g + 1] >> 5) & 0x03FC03FCu;  // 4e of elements 4g+2, 4g+3
    const uint32_t t0 = lds_u32_off<0>(base + (f0 & 0xFFFFu));
    const uint32_t t1 = lds_u32_off<1024>(base + (f0 >> 16));
    const uint32_t t2 = lds_u32_off<2048>(base + (f1 & 0xFFFFu));
    const uint32_t t3 = lds_u32_off<3072>(base + (f1 >> 16));
    return sum4(t0, t1, t2, t3, one);
  }
}

// E5M2 sign|mantissa 3-bit symbols of group g as a 12-bit little-endian group
// (formats.py:184-189 on a = sign<<2 | mantissa, formats.py:123-125): the
// six bits of elements (0,1) gather at bits 0-5 and of (2,3) at bits 16-21.
// The same 12-bit group at bits 20-31 of the result (bits 0-19 are junk),
// gathered by two multiplies on the FMA pipe: after masking the sign and
// mantissa bits of bytes 0-1 (resp. 2-3), x 1057 (= 1 + 2^5 + 2^10) moves
// every wanted bit to its place at once — all partial products land on
// distinct bits, so no carries — and a bit-select merges the halves.
// k_lo = 1057 << 10 and k_hi = 1057 are kernel arguments so ptxas keeps the
// multiplies (it would expand a literal into ALU shifts and adds).
__device__ __forceinline__ uint32_t e5m2_sm_hi(uint32_t x, uint32_t k_lo, uint32_t k_hi) {
  const uint32_t lo = w_mad(x & 0x00008383u, k_lo, 0u);  // symbols 0,1 -> bits 20-25
  const uint32_t hi = w_mad(x & 0x83830000u, k_hi, 0u);  // symbols 2,3 -> bits 26-31
  return bitselect(lo, hi, 0x03F00000u);
}

__device__ __forceinline__ uint32_t e5m2_sm12(uint32_t x) {
  const uint32_t u = (x & 0x00030003u) | ((x >> 5) & 0x001C001Cu) | ((x >> 10) & 0x00200020u);
  return (u | (u >> 10)) & 0xFFFu;
}

template <int FMT>
__device__ __forceinline__ uint32_t raw_exponent(uint32_t word) {
  if constexpr (FMT == SZ_BF16) return (word >> 7) & 0xFF;
  else if constexpr (FMT == SZ_E5M2) return (word >> 2) & 0x1F;
  else return (word >> 3) & 0x0F;
}

// Dense transform of one 32-byte slot; returns the slot's escape bitmask.
// TAIL=false is the steady-state path (slot fully inside N, stores at the
// precomputed slot addresses); TAIL=true handles the ragged last slots.
template <int FMT, int CB, bool TAIL>
__device__ __forceinline__ uint32_t encode_slot(const uint32_t (&x)[8], const uint8_t* lut,
                                                int nv, uint8_t* cdst, uint8_t* sdst,
                                                const EncodeArgs& a, uint64_t e0) {
  constexpr int EPV = kEpv<FMT>;
  constexpr int G = EPV / 4;
  constexpr int SMB = Fmt<FMT>::kSmBits;
  constexpr int CBYTES = EPV * CB / 8;
  constexpr int SBYTES = EPV * SMB / 8;
  constexpr int CWORDS = (CBYTES + 3) / 4;
  constexpr int SWORDS = (SBYTES + 3) / 4;
  const uint32_t base = smem_addr(lut);  // the T4 tables (see t4_group)
  uint32_t r[G];
  uint32_t any = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    r[g] = t4_group<FMT>(x, g, base, a.lut_stride, a.one);
    if (TAIL && nv < EPV) {  // tail slot: no codes or flags beyond N (x is 0 there)
      const int v = min(max(nv - 4 * g, 0), 4);
      r[g] &= v >= 4 ? 0xFFFFFFFFu
                     : (((1u << (CB * v)) - 1u) | (((1u << v) - 1u) << 16) |
                        (((1u << (3 * v)) - 1u) << 20));
    }
    any |= r[g];
  }
  uint32_t fm = 0;
  if (any & 0x000F0000u) {
#pragma unroll
    for (int g = 0; g < G; ++g) fm |= ((r[g] >> 16) & 0xFu) << (4 * g);
  }
  uint32_t cw[CWORDS], sw[SWORDS];
  if constexpr (CB == 4) {
#pragma unroll
    for (int i = 0; i < CWORDS; ++i) cw[i] = __byte_perm(r[2 * i], r[2 * i + 1], 0x5410);
  } else {
    uint32_t grp[G];
#pragma unroll
    for (int g = 0; g < G; ++g) grp[g] = r[g] & 0xFFFu;
    concat_groups<G, 12>(grp, cw);
  }
  if constexpr (FMT == SZ_E4M3) {
    uint32_t grp[G];
#pragma unroll
    for (int g = 0; g < G; ++g)
      grp[g] = pack_nib4(((x[g] >> 4) & 0x08080808u) | (x[g] & 0x07070707u));
    concat_groups<G, 16>(grp, sw);
  } else if constexpr (FMT == SZ_BF16) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t lo4 = __byte_perm(x[2 * g], x[2 * g + 1], 0x6420);
      const uint32_t hi4 = __byte_perm(x[2 * g], x[2 * g + 1], 0x7531);
      sw[g] = bitselect(hi4, lo4, 0x80808080u);
    }
  } else {
    // 12-bit SM groups in bits 20-31: of each lookup result (full-byte
    // tables) or of e5m2_sm_hi
    uint32_t h[G];
#pragma unroll
    for (int g = 0; g < G; ++g) h[g] = kE5FullByte ? r[g] : e5m2_sm_hi(x[g], a.k_lo, a.k_hi);
    sw[0] = (h[0] >> 20) | ((h[1] >> 8) & 0x00FFF000u) | ((h[2] << 4) & 0xFF000000u);
    sw[1] = (h[2] >> 28) | ((h[3] >> 16) & 0x0000FFF0u) | ((h[4] >> 4) & 0x0FFF0000u) |
            ((h[5] << 8) & 0xF0000000u);
    sw[2] = (h[5] >> 24) | ((h[6] >> 12) & 0x000FFF00u) | (h[7] & 0xFFF00000u);
  }
  if (!TAIL || nv == EPV) {
    st_packed<CBYTES>(cdst, cw);
    st_packed<SBYTES>(sdst, sw);
  } else if (nv > 0) {
    st_bytes_clipped<CBYTES>(a.codes, e0 * CB / 8, cw, a.codes_len);
    st_bytes_clipped<SBYTES>(a.sm, e0 * SMB / 8, sw, a.sm_len);
  }
  return fm;

}

// Position of element `idx` in the escape-position stream (codec.py:289-295).
template <int POSB>
__device__ __forceinline__ void put_position(uint8_t* base, uint64_t i, uint64_t idx,
                                             uint32_t chunk, int32_t chunk_shift) {
  if constexpr (POSB == 4) {
    reinterpret_cast<uint32_t*>(base)[i] = static_cast<uint32_t>(idx);
  } else if constexpr (POSB == 2 || POSB == 1) {
    const uint64_t pos = chunk_shift >= 0 ? (idx & (chunk - 1)) : (idx % chunk);
    if constexpr (POSB == 2) reinterpret_cast<uint16_t*>(base)[i] = static_cast<uint16_t>(pos);
    else base[i] = static_cast<uint8_t>(pos);
  }
}

// 2-D tensor TMA: one 128 B x 256-row box (one 32 KiB tile) into shared
// memory with the 128B swizzle (16-byte chunk c of row r lands at chunk
// c ^ (r & 7)), completion counted on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x,
                                            int32_t y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

template <int FMT, int CB, int POSB>
__global__ void __launch_bounds__(kEncThreads<FMT, CB>, 1)
    encode_tiles(const __grid_constant__ sz_params p, const EncodeArgs a,
                 const __grid_constant__ CUtensorMap tmap) {
  constexpr int EPV = kEpv<FMT>;
  constexpr int WB = Fmt<FMT>::kWordBytes;
  constexpr uint64_t TILE = static_cast<uint64_t>(kEncSlots) * EPV;
  constexpr int SMB = Fmt<FMT>::kSmBits;
  constexpr int CBYTES = EPV * CB / 8;
  constexpr int SBYTES = EPV * SMB / 8;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int NW = kWriterWarps<FMT, CB>;
  constexpr int NT = kEncThreads<FMT, CB>;
  constexpr int QS = kScanSlots<FMT, CB>;
  constexpr int VCAP = kEscValCap<FMT>;
  EncSmem<FMT, CB>& S = *reinterpret_cast<EncSmem<FMT, CB>*>(
      smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;
  // T4 lane tables (t4_group), 1 KiB aligned: PRMT-built addresses
  constexpr int TE = kT4Entries<FMT>;
  __shared__ __align__(1024) uint32_t s_tab[4 * TE];
  const uint8_t* s_lut = reinterpret_cast<const uint8_t*>(s_tab);
  for (int i = tid; i < 4 * TE; i += NT) {
    const int k = i / TE, e = i % TE;
    if constexpr (FMT == SZ_E5M2 && kE5FullByte) {  // e is the whole byte here
      const uint32_t m = p.enc_lut[(e >> 2) & 31];
      const uint32_t a = ((e >> 5) & 4u) | (e & 3u);
      s_tab[i] = ((m & ((1u << CB) - 1u)) << (CB * k)) | (((m >> 4) & 1u) << (16 + k)) |
                 (a << (20 + 3 * k));
    } else {
      const uint32_t m = p.enc_lut[e];
      s_tab[i] = ((m & ((1u << CB) - 1u)) << (CB * k)) | (((m >> 4) & 1u) << (16 + k));
    }
  }
  pdl_trigger();
  pdl_wait();  // (the tables above come from kernel parameters only)
  if (blockIdx.x == 0 && tid == 0) *a.base_snapshot = a.escape_base ? *a.escape_base : 0;
  if (tid == 0) {
    for (int s = 0; s < kEncInStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.in_empty[s], kEncDense);
    }
    for (int q = 0; q < QS; ++q) {
      mbar_init(&S.computed[q], kEncDense);
      mbar_init(&S.scan_empty[q], 32);  // every writer lane arrives
      S.esc_n[q] = 0;
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      long long t_in = 0, t_scan = 0;
      // Paged input: the tile is claimed one iteration ahead and its first
      // segment address loaded before the stage waits, so neither the
      // claim's atomic nor the segment-table load sits between a free stage
      // and its TMA.
      const bool ahead = a.seg_addrs != nullptr;
      uint64_t next = ahead ? atomicAdd(a.tile_counter, 1ull) : 0;
      for (uint32_t it = 0;; ++it) {
        const uint32_t s = it % kEncInStages, sph = (it / kEncInStages) & 1;
        const uint32_t q = it % QS, qph = (it / QS) & 1;
        uint64_t seg_first = 0;
        if (ahead && next < a.num_tiles)
          seg_first = __ldg(a.seg_addrs + ((next * TILE * WB) >> a.seg_shift));
        const long long c0 = SZ_CLOCK();
        mbar_wait(&S.in_empty[s], sph ^ 1);
        const long long c1 = SZ_CLOCK();
        mbar_wait(&S.scan_empty[q], qph ^ 1);
        t_in += c1 - c0;
        t_scan += SZ_CLOCK() - c1;
        uint64_t tile;
        if (ahead) {
          tile = next;
          if (tile < a.num_tiles) next = atomicAdd(a.tile_counter, 1ull);
        } else {
          tile = atomicAdd(a.tile_counter, 1ull);
        }
        if (tile >= a.num_tiles) {
          // end markers in this slot and the next NW-1 (one per
          // writer residue class); the dense warps relay them (computed)
          S.meta[q] = ~0ull;
          for (uint32_t k = 1; k < NW; ++k) {
            const uint32_t qk = (it + k) % QS, pk = ((it + k) / QS) & 1;
            mbar_wait(&S.scan_empty[qk], pk ^ 1);
            S.meta[qk] = ~0ull;
          }
          mbar_arrive(&S.full[s]);
          break;
        }
        S.meta[q] = tile;
        const uint64_t e0 = tile * TILE;
        const uint32_t full_slots = static_cast<uint32_t>(min(n - e0, TILE) / EPV);
        const uint32_t bytes = full_slots * 32;
        if (a.seg_tmap && e0 + TILE <= n) {
          // paged KV through the VA-window tensor map: one swizzled box per
          // segment (or per tile, for segments >= a tile)
          mbar_arrive_tx(&S.full[s], kEncTileBytes);
          const uint64_t b0 = e0 * WB, seg_mask = (1ull << a.seg_shift) - 1;
          const uint32_t piece = static_cast<uint32_t>(
              min(static_cast<uint64_t>(kEncTileBytes), seg_mask + 1));
          for (uint32_t o = 0; o < static_cast<uint32_t>(kEncTileBytes); o += piece) {
            const uint64_t g = b0 + o;
            const uint64_t addr =
                (o == 0 ? seg_first : __ldg(a.seg_addrs + (g >> a.seg_shift))) + (g & seg_mask);
            tma_load_2d(S.in[s] + o, &tmap, 0, static_cast<int32_t>((addr - a.seg_va_lo) >> 7),
                        &S.full[s]);
          }
        } else if (a.seg_addrs) {
          // paged KV: one bulk copy per (tile ∩ segment) piece, straight from
          // the cache blocks — no gather pass through HBM
          if (bytes) mbar_arrive_tx(&S.full[s], bytes);
          else mbar_arrive(&S.full[s]);
          const uint64_t b0 = e0 * WB, seg_mask = (1ull << a.seg_shift) - 1;
          for (uint32_t o = 0; o < bytes;) {
            const uint64_t g = b0 + o;
            const uint32_t len = static_cast<uint32_t>(
                min(static_cast<uint64_t>(bytes - o), (seg_mask + 1) - (g & seg_mask)));
            const uint8_t* src = reinterpret_cast<const uint8_t*>(
                                     __ldg(a.seg_addrs + (g >> a.seg_shift))) + (g & seg_mask);
            tma_load_1d(S.in[s] + o, src, len, &S.full[s]);
            o += len;
          }
        } else if (a.use_tmap && e0 + TILE <= n) {
          mbar_arrive_tx(&S.full[s], kEncTileBytes);
          tma_load_2d(S.in[s], &tmap, 0, static_cast<int32_t>(tile * (kEncTileBytes / 128)),
                      &S.full[s]);
        } else if (bytes) {
          mbar_arrive_tx(&S.full[s], bytes);
          tma_load_1d(S.in[s], a.words + e0 * WB, bytes, &S.full[s]);
        } else {
          mbar_arrive(&S.full[s]);
        }
      }
      if (a.dbg) {
        atomicAdd(&a.dbg[6], static_cast<unsigned long long>(t_in));
        atomicAdd(&a.dbg[7], static_cast<unsigned long long>(t_scan));
      }
    }
    return;
  }

  if (warp < kEncDenseWarps) {
    // ------------------------------------------------------------ dense warps
    long long t_wait = 0, t_work = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it % kEncInStages, sph = (it / kEncInStages) & 1;
      const uint32_t q = it % QS, qph = (it / QS) & 1;
      const long long c0 = SZ_CLOCK();
      mbar_wait(&S.full[s], sph);
      // direct ordering after the writer's release of this scan slot (also
      // implied through the producer; re-checked at no cost)
      mbar_wait(&S.scan_empty[q], qph ^ 1);
      const long long c1 = SZ_CLOCK();
      t_wait += c1 - c0;
      const uint64_t tile = S.meta[q];
      if (tile == ~0ull) {
        for (uint32_t k = 0; k < NW; ++k)
          mbar_arrive(&S.computed[(it + k) % QS]);
        break;
      }
      const uint64_t tile_e0 = tile * TILE;
      const bool tail_tile = tile_e0 + TILE > n;
      uint8_t* const ctile = a.codes + tile_e0 * CB / 8;
      uint8_t* const stile = a.sm + tile_e0 * SMB / 8;
      uint32_t x[kEncItems][8];
      int nv[kEncItems];
      // (steady state) byte offsets of the slot's two 16-byte halves in its
      // 128-byte stage row; the escape loop below re-reads words from there
      const uint32_t rsw = (tid >> 2) & 7, cc0 = 2 * (tid & 3);
      const uint32_t off0 = a.use_tmap ? ((cc0 ^ rsw) << 4) : (tid & 3) * 32;
      const uint32_t off1 = a.use_tmap ? (((cc0 + 1) ^ rsw) << 4) : (tid & 3) * 32 + 16;
      if (!tail_tile) {
        // steady state: every slot is full and in the TMA stage.  Slot
        // i*512 + tid is row (slot >> 2) of 128 B, 16-byte chunks 2(tid&3) and
        // 2(tid&3)+1; with the swizzle they sit at chunk ^ (row & 7), and
        // row & 7 = (tid >> 2) & 7 — per-thread constants.  A quarter-warp then
        // reads 8 distinct chunks of 2 rows: no bank conflicts (the linear
        // layout's 32-byte stride made every read 2-way conflicted).
#pragma unroll
        for (int i = 0; i < kEncItems; ++i) {
          const uint8_t* row = S.in[s] + (i * kEncDense + tid) / 4 * 128;
          const uint4 v0 = *reinterpret_cast<const uint4*>(row + off0);
          const uint4 v1 = *reinterpret_cast<const uint4*>(row + off1);
          x[i][0] = v0.x; x[i][1] = v0.y; x[i][2] = v0.z; x[i][3] = v0.w;
          x[i][4] = v1.x; x[i][5] = v1.y; x[i][6] = v1.z; x[i][7] = v1.w;
          nv[i] = EPV;
        }
      } else {
#pragma unroll
        for (int i = 0; i < kEncItems; ++i) {
          const int slot = i * kEncDense + tid;
          const uint64_t e0 = tile_e0 + static_cast<uint64_t>(slot) * EPV;
          nv[i] = e0 + EPV <= n ? EPV : (e0 < n ? static_cast<int>(n - e0) : 0);
          if (nv[i] == EPV) {
            const uint4* src = reinterpret_cast<const uint4*>(S.in[s] + slot * 32);
            const uint4 v0 = src[0], v1 = src[1];
            x[i][0] = v0.x; x[i][1] = v0.y; x[i][2] = v0.z; x[i][3] = v0.w;
            x[i][4] = v1.x; x[i][5] = v1.y; x[i][6] = v1.z; x[i][7] = v1.w;
          } else {
            ld_bytes_clipped<32>(a.words, e0 * WB, x[i], nv[i] > 0 ? n * WB : 0);
          }
        }
      }
      uint32_t fms[kEncItems];
#pragma unroll
      for (int i = 0; i < kEncItems; ++i) {
        const int slot = i * kEncDense + tid;
        uint32_t fm;
        if (!tail_tile) {
          fm = encode_slot<FMT, CB, false>(x[i], s_lut, EPV, ctile + slot * CBYTES,
                                           stile + slot * SBYTES, a, 0);
        } else {
          fm = encode_slot<FMT, CB, true>(x[i], s_lut, nv[i], ctile + slot * CBYTES,
                                          stile + slot * SBYTES, a,
                                          tile_e0 + static_cast<uint64_t>(slot) * EPV);
        }
        S.fmask[q][fsw(slot)] = fm;
        fms[i] = fm;
      }
      // input stage free: the producer may refill it (a thread with escapes
      // holds it through its escape loop, which re-reads the words there)
      const bool any_esc = (fms[0] | fms[1]) != 0u;
      static_assert(kEncItems == 2, "any_esc covers two items");
      if (!any_esc) mbar_arrive(&S.in_empty[s]);
#pragma unroll
      for (int i = 0; i < kEncItems; ++i) {
        const int slot = i * kEncDense + tid;
        const uint32_t fm = fms[i];
        if (fm) {  // append this slot's escape records for the writer
          const uint32_t c = static_cast<uint32_t>(__popc(fm));
          uint32_t r = atomicAdd(&S.esc_n[q], c);
          // a tile past VCAP is re-derived whole by K2c: none of its
          // records is used, so stop writing them
          uint32_t f = r + c <= VCAP ? fm : 0u;
          const uint8_t* row = S.in[s] + (i * kEncDense + tid) / 4 * 128;
          while (f) {  // compact loop
            const int j = __ffs(f) - 1;
            f &= f - 1;
            uint32_t word;
            if (!tail_tile) {  // the word again from the (still held) input stage
              const uint32_t bo = static_cast<uint32_t>(j) * WB;
              const uint8_t* wp = row + ((bo >> 4) ? off1 : off0) + (bo & 15u);
              if constexpr (WB == 2) word = *reinterpret_cast<const uint16_t*>(wp);
              else word = *wp;
            } else {  // x[] read through selects (no local memory)
              if constexpr (WB == 2) word = (pick<8>(x[i], j >> 1) >> (16 * (j & 1))) & 0xFFFFu;
              else word = (pick<8>(x[i], j >> 2) >> (8 * (j & 3))) & 0xFFu;
            }
            S.esc_idx[q][r] = static_cast<uint16_t>(slot * EPV + j);
            S.esc_val[q][r++] = static_cast<uint8_t>(raw_exponent<FMT>(word));
          }
        }
      }
      if (any_esc) mbar_arrive(&S.in_empty[s]);
      mbar_arrive(&S.computed[q]);
      t_work += SZ_CLOCK() - c1;
    }
    if (a.dbg && lane == 0) {
      atomicAdd(&a.dbg[0], static_cast<unsigned long long>(t_wait));
      atomicAdd(&a.dbg[1], static_cast<unsigned long long>(t_work));
    }
    return;
  }

  // ---------------------------------------------------------------- writer warps
  constexpr int SPL = kEncSlots / 32;  // 32 consecutive slots per lane
  const int ww = warp - kWriterWarp0;  // owns iterations it == ww (mod NW)
  uint16_t* sp = S.slot_pref[ww];
  const uint32_t key = fsw_key(lane);  // this lane's slots: lane*SPL + (j ^ key)
  long long t_wait = 0, t_work = 0;
  for (uint32_t it = ww;; it += NW) {
    const uint32_t q = it % QS, qph = (it / QS) & 1;
    const long long c0 = SZ_CLOCK();
    mbar_wait(&S.computed[q], qph);
    const long long c1 = SZ_CLOCK();
    t_wait += c1 - c0;
    const uint64_t tile = S.meta[q];
    if (tile == ~0ull) break;
    const uint64_t tile_e0 = tile * TILE;

    const uint32_t* fm = &S.fmask[q][lane * SPL];  // slot lane*SPL + j at fm[j ^ key]
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < SPL; j += 4) {  // (4 masks of one aligned group, permuted)
      const uint4 v = *reinterpret_cast<const uint4*>(fm + (j ^ (key & ~3u)));
      cnt += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    const uint32_t excl_lane = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0) a.tile_esc[tile] = total;

    if (a.counts_mode == 1) {
      // chunks tile the CTA tile (power-of-two chunk): count straight from the
      // lane scan
      const uint32_t spc = a.chunk / EPV;                 // slots per chunk
      const uint64_t k_base = tile_e0 / a.chunk;
      if (spc >= SPL) {
        const uint32_t L = spc / SPL;                     // lanes per chunk
        const uint32_t first = lane & ~(L - 1);
        const uint32_t start_excl = __shfl_sync(0xffffffffu, excl_lane, first);
        const uint64_t k = k_base + lane / L;
        if ((lane & (L - 1)) == L - 1 && k < a.n_chunks) a.counts[k] = incl - start_excl;
      } else {
        const uint32_t per_lane = SPL / spc;
        for (uint32_t c = 0; c < per_lane; ++c) {
          uint32_t sum = 0;
          for (uint32_t j = c * spc; j < (c + 1) * spc; ++j) sum += __popc(fm[j ^ key]);
          const uint64_t k = k_base + lane * per_lane + c;
          if (k < a.n_chunks) a.counts[k] = sum;
        }
      }
    }
    if (a.counts_mode == 2 && total) {
      const uint64_t last = min(tile_e0 + TILE, n) - 1;
      const uint64_t k0 = tile_e0 / a.chunk;
      if (k0 == last / a.chunk) {
        if (lane == 0) atomicAdd(&a.counts[k0], total);
      } else {
        for (int j = 0; j < SPL; ++j) {
          uint32_t m = fm[j ^ key];
          const uint64_t e0 = tile_e0 + static_cast<uint64_t>(lane * SPL + j) * EPV;
          while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            atomicAdd(&a.counts[(e0 + b) / a.chunk], 1u);
          }
        }
      }
    }

    // The tile's escape records into its scratch slot in ascending element
    // order: per-slot prefixes from the lane scan, then consecutive lanes on
    // consecutive records (balanced whatever the escapes' clustering), each
    // record's rank = its slot's prefix + the escapes below it in the slot.
    if (total && total <= VCAP) {
      uint32_t run = excl_lane;
      for (int j = 0; j < SPL; ++j) {
        sp[lane * SPL + (j ^ key)] = run;
        run += __popc(fm[j ^ key]);
      }
      __syncwarp();
      uint8_t* const sval = a.scr_val + tile * kTileCap<FMT>;
      uint8_t* const spos = a.scr_pos + tile * kTileCap<FMT> * (POSB ? POSB : 1);
      // positions in 32-bit arithmetic: chunk-relative = (tile start mod
      // chunk + local) mod chunk; abs32 = tile start + local (n < 2^32)
      const uint32_t pbase = POSB == 4 ? static_cast<uint32_t>(tile_e0)
                             : static_cast<uint32_t>(a.chunk_shift >= 0
                                                         ? tile_e0 & (a.chunk - 1)
                                                         : tile_e0 % a.chunk);
      const uint32_t* const fmq = S.fmask[q];
      const uint16_t* const idq = S.esc_idx[q];
      const uint8_t* const vaq = S.esc_val[q];
#pragma unroll 4
      for (uint32_t r = lane; r < total; r += 32) {
        const uint32_t local = idq[r];
        const uint32_t slot = local / EPV, b = local % EPV;
        const uint32_t fs = fsw(slot);
        const uint32_t rank = sp[fs] + __popc(fmq[fs] & ((1u << b) - 1u));
        sval[rank] = vaq[r];
        if constexpr (POSB == 4) {
          reinterpret_cast<uint32_t*>(spos)[rank] = pbase + local;
        } else if constexpr (POSB == 1 || POSB == 2) {
          uint32_t pos = pbase + local;
          pos = a.chunk_shift >= 0 ? (pos & (a.chunk - 1)) : (pos % a.chunk);
          if constexpr (POSB == 2) reinterpret_cast<uint16_t*>(spos)[rank] = static_cast<uint16_t>(pos);
          else spos[rank] = static_cast<uint8_t>(pos);
        }
      }
    }
    __syncwarp();
    if (lane == 0) S.esc_n[q] = 0;
    __syncwarp();
    mbar_arrive(&S.scan_empty[q]);
    t_work += SZ_CLOCK() - c1;
  }
  if (a.dbg && lane == 0) {
    atomicAdd(&a.dbg[2], static_cast<unsigned long long>(t_wait));
    atomicAdd(&a.dbg[3], static_cast<unsigned long long>(t_work));
  }
}

// ------------------------------------------------------------------ K2b
struct GatherArgs {
  const uint8_t* words;
  const uint64_t* seg_addrs;  // segmented input (or null)
  uint32_t seg_shift;
  uint64_t n;
  const uint32_t* tile_esc;
  const uint8_t* scr_pos;
  const uint8_t* scr_val;
  uint64_t num_tiles;
  uint64_t tile_elems;
  uint8_t* positions;
  uint8_t* values;
  uint64_t capacity;
  uint64_t* n_escapes;
  const uint64_t* tile_pref;      // exclusive escape prefix per tile (+ total), from the scan
  uint64_t* scan_states;          // (the scan's look-back states and ticket, for its launch)
  unsigned long long* scan_counter;
  unsigned long long* counter;
  uint64_t num_groups;
  uint32_t chunk;
  int32_t chunk_shift;
  const uint64_t* base_snapshot;  // append offset captured by K2a
  uint64_t* escape_base;          // append mode: advanced by this call's M
  // escape-heavy tiles (more escapes than a scratch slot): K2b lists them
  // with their first ordinal; K2c re-derives them, one CTA per tile
  uint32_t* heavy_list;
  uint64_t* heavy_pref;           // per listed tile: first global ordinal
  unsigned int* heavy_count;
  uint32_t split;                 // CTAs per group (record moves split R ways)
};

// Warp copy of nbytes from a 4-byte-aligned source to an arbitrary
// destination: destination word w holds source bytes [4w - sh, 4w - sh + 4),
// sh = the destination's misalignment, built from source words w-1 (from the
// neighbouring lane) and w by one funnel shift; the partial first / last
// words are written bytewise (their other bytes belong to neighbouring runs).
__device__ __forceinline__ void warp_copy_bytes(uint8_t* dst, const uint8_t* src,
                                                uint32_t nbytes, int lane) {
  if (nbytes == 0) return;
  const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 3u);
  uint8_t* const d0 = dst - sh;
  const uint32_t* const sw = reinterpret_cast<const uint32_t*>(src);
  const uint32_t nwords = (sh + nbytes + 3) >> 2;
  constexpr int U = 4;   // rounds per step: all their loads in flight first
  uint32_t carry = 0;    // source word (base - 1), from the previous round's lane 31
  for (uint32_t base = 0; base < nwords; base += 32 * U) {
    uint32_t hi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w = base + 32 * u + lane;
      hi[u] = 4 * w < nbytes ? __ldg(sw + w) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w = base + 32 * u + lane;
      uint32_t lo = __shfl_up_sync(0xffffffffu, hi[u], 1);
      if (lane == 0) lo = carry;
      carry = __shfl_sync(0xffffffffu, hi[u], 31);
      if (w < nwords) {
        const uint32_t v = sh ? __funnelshift_l(lo, hi[u], 8 * sh) : hi[u];
        // bytes of this word inside [sh, sh + nbytes) of the destination span
        const uint32_t b0 = 4 * w, b1 = b0 + 4;
        if (b0 >= sh && b1 <= sh + nbytes) {
          *reinterpret_cast<uint32_t*>(d0 + b0) = v;
        } else {
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i)
            if (b0 + i >= sh && b0 + i < sh + nbytes) d0[b0 + i] = static_cast<uint8_t>(v >> (8 * i));
        }
      }
    }
  }
}

// Tiles per CTA: 256 (8 per lane in the scan) keeps the look-back chain
// short — K2b is latency-bound, so fewer, fatter CTAs win.
constexpr int kGatherTiles = 256;
constexpr int kGatherUnroll = 4;
#ifdef SZ_NO_SPARSE2
constexpr bool kSparse2 = false;
#else
constexpr bool kSparse2 = true;
#endif
static_assert(kGatherTiles == 256, "escape_gather's search does exactly 8 halvings");

template <int FMT, int POSB>
__global__ void __launch_bounds__(kThreads)
    escape_gather(const __grid_constant__ sz_params p, const GatherArgs a) {
  __shared__ uint64_t tpref[kGatherTiles];
  __shared__ uint32_t tcnt[kGatherTiles];
  // group-relative prefix of the records K2b moves (regular tiles only; an
  // escape-heavy tile counts 0 here, K2c writes its records)
  __shared__ uint32_t rpref[kGatherTiles + 1];
  __shared__ unsigned long long s_group;
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Tickets: group = ticket / R, part = ticket % R; part p of a group moves
  // its share of the group's records (escape-dense inputs get R x the CTAs).
  if (tid == 0) s_group = atomicAdd(a.counter, 1ull);
  __syncthreads();
  const uint64_t group = s_group / a.split;
  const uint32_t part = static_cast<uint32_t>(s_group % a.split);
  const uint64_t t0 = group * kGatherTiles;
  if (warp == 0) {
    // the group's first ordinal (tile-prefix scan) and the append base,
    // loaded together with the tile counts: one memory latency, not two
    const uint64_t ex = __ldg(a.tile_pref + t0);
    const uint64_t base = *a.base_snapshot;
    // each lane owns kTilesPerLane consecutive tiles of the group
    constexpr int kTilesPerLane = kGatherTiles / 32;
    constexpr uint32_t CAP = kTileCap<FMT>;
    uint32_t c[kTilesPerLane];
    uint64_t lsum = 0;
    uint32_t rsum = 0;
#pragma unroll
    for (int j = 0; j < kTilesPerLane; ++j) {
      const uint64_t t = t0 + lane * kTilesPerLane + j;
      c[j] = t < a.num_tiles ? a.tile_esc[t] : 0u;
      lsum += c[j];
      rsum += c[j] <= CAP ? c[j] : 0u;
    }
    uint64_t incl = lsum;
    uint32_t rincl = rsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t o = __shfl_up_sync(0xffffffffu, incl, d);
      const uint32_t ro = __shfl_up_sync(0xffffffffu, rincl, d);
      if (lane >= d) { incl += o; rincl += ro; }
    }
    {
      uint32_t rrun = rincl - rsum;
#pragma unroll
      for (int j = 0; j < kTilesPerLane; ++j) {
        rpref[lane * kTilesPerLane + j] = rrun;
        rrun += c[j] <= CAP ? c[j] : 0u;
      }
      if (lane == 31) rpref[kGatherTiles] = rincl;
    }
    uint64_t run = base + ex + incl - lsum;
#pragma unroll
    for (int j = 0; j < kTilesPerLane; ++j) {
      tpref[lane * kTilesPerLane + j] = run;
      tcnt[lane * kTilesPerLane + j] = c[j];
      run += c[j];
    }
    if (lane == 0 && part == 0 && group == a.num_groups - 1) {
      const uint64_t total = a.tile_pref[a.num_tiles];
      *a.n_escapes = total;
      if (a.escape_base) *a.escape_base = base + total;
    }
  }
  __syncthreads();
  // Flat pass over every record of the group's regular tiles: thread t moves
  // records t, t+256, ... (tile found by a search over the regular-record
  // prefixes), so all loads of the group are in flight at once.  Heavy
  // tiles' records are not visited at all (an all-heavy input leaves K2b
  // only its scan and the listing).
  // Sparse groups (<= 32 records per tile on average) move tile by tile
  // instead: a warp takes 4 tiles at a time, lane r moves record r of each —
  // no per-record search (the flat pass's binary search made K2b
  // instruction-bound at realistic escape rates).
  auto move = [&](uint64_t src, uint64_t dst) {
    a.values[dst] = a.scr_val[src];
    if constexpr (POSB == 1) a.positions[dst] = a.scr_pos[src];
    else if constexpr (POSB == 2)
      reinterpret_cast<uint16_t*>(a.positions)[dst] = reinterpret_cast<const uint16_t*>(a.scr_pos)[src];
    else if constexpr (POSB == 4)
      reinterpret_cast<uint32_t*>(a.positions)[dst] = reinterpret_cast<const uint32_t*>(a.scr_pos)[src];
  };
  // RPL records per lane (lane + 32j of each of the warp's TU tiles): all
  // TU x RPL loads in flight before any store.
  auto sparse = [&](auto rpl_c) {
    constexpr int RPL = decltype(rpl_c)::value;
    const int k_lo = static_cast<int>(kGatherTiles * part / a.split);
    const int k_hi = static_cast<int>(kGatherTiles * (part + 1) / a.split);
    constexpr int TU = 4;
    for (int k0 = k_lo + warp * TU; k0 < k_hi; k0 += kWarps * TU) {
      uint64_t src[TU], dst[TU];
      uint32_t val[TU][RPL], pos[TU][RPL], cnt[TU];
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const int k = k0 + u;
        cnt[u] = k < k_hi ? tcnt[k] : 0u;   // 0 past the last tile of the stream
        if (cnt[u] > kTileCap<FMT>) cnt[u] = 0;  // heavy: K2c's
        src[u] = (t0 + k) * kTileCap<FMT> + lane;
        dst[u] = (k < k_hi ? tpref[k] : 0) + lane;
      }
      auto live = [&](int u, int j) {
        return lane + 32u * j < cnt[u] && dst[u] + 32u * j < a.capacity;
      };
#pragma unroll
      for (int u = 0; u < TU; ++u)
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          if (!live(u, j)) continue;
          const uint64_t sj = src[u] + 32u * j;
          val[u][j] = __ldg(a.scr_val + sj);
          if constexpr (POSB == 1) pos[u][j] = __ldg(a.scr_pos + sj);
          else if constexpr (POSB == 2) pos[u][j] = __ldg(reinterpret_cast<const uint16_t*>(a.scr_pos) + sj);
          else if constexpr (POSB == 4) pos[u][j] = __ldg(reinterpret_cast<const uint32_t*>(a.scr_pos) + sj);
        }
#pragma unroll
      for (int u = 0; u < TU; ++u)
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          if (!live(u, j)) continue;
          const uint64_t dj = dst[u] + 32u * j;
          a.values[dj] = static_cast<uint8_t>(val[u][j]);
          if constexpr (POSB == 1) a.positions[dj] = static_cast<uint8_t>(pos[u][j]);
          else if constexpr (POSB == 2) reinterpret_cast<uint16_t*>(a.positions)[dj] = static_cast<uint16_t>(pos[u][j]);
          else if constexpr (POSB == 4) reinterpret_cast<uint32_t*>(a.positions)[dj] = pos[u][j];
        }
#pragma unroll
      for (int u = 0; u < TU; ++u)  // tiles with more than 32 x RPL records (rare here)
        for (uint32_t r = lane + 32 * RPL; r < cnt[u]; r += 32)
          if (dst[u] - lane + r < a.capacity) move(src[u] - lane + r, dst[u] - lane + r);
    }
  };
  if (rpref[kGatherTiles] <= 32u * kGatherTiles) {
    sparse(std::integral_constant<int, 1>{});
  } else if (kSparse2 && rpref[kGatherTiles] <= 64u * kGatherTiles) {
    // realistic FP8 streams (32K-element tiles, ~52 records per tile at
    // eps 0.16%): two records per lane instead of the flat pass's search
    sparse(std::integral_constant<int, 2>{});
  } else if (rpref[kGatherTiles] > 512u * kGatherTiles) {
    // Escape-dense groups (> 512 records per tile on average): a tile's records are one contiguous run in its
    // scratch slot and one contiguous run in each output section, so a warp
    // moves a whole (tile, section) run as 32-bit words realigned with a
    // funnel shift (the scratch slot is 16-byte aligned, the destination
    // arbitrary): coalesced 128-byte warp accesses instead of a byte or u16
    // per record, and no per-record tile search.
    const int k_lo = static_cast<int>(kGatherTiles * part / a.split);
    const int k_hi = static_cast<int>(kGatherTiles * (part + 1) / a.split);
    const int items = 2 * (k_hi - k_lo);   // (tile, values | positions)
    for (int it = warp; it < items; it += kWarps) {
      const int k = k_lo + (it >> 1);
      const uint32_t cnt = tcnt[k];
      if (cnt == 0 || cnt > kTileCap<FMT>) continue;   // empty, or heavy (K2c's)
      const uint64_t dst = tpref[k];
      if (dst >= a.capacity) continue;
      const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(cnt), a.capacity - dst));
      const uint64_t src = (t0 + k) * kTileCap<FMT>;
      if ((it & 1) == 0)
        warp_copy_bytes(a.values + dst, a.scr_val + src, n, lane);
      else if constexpr (POSB != 0)
        warp_copy_bytes(a.positions + dst * POSB, a.scr_pos + src * POSB, n * POSB, lane);
    }
  } else {
    const uint64_t g_all = rpref[kGatherTiles];
    const uint64_t g_lo = g_all * part / a.split, g_hi = g_all * (part + 1) / a.split;
    const uint64_t g_total = g_hi - g_lo;
    // kGatherUnroll records per thread per round: all loads are issued before
    // any store, so the round costs one memory latency, not kGatherUnroll.
    constexpr int U = kGatherUnroll;
    // r's tile = the last k with rpref[k] <= r.  A thread's records only
    // increase (by 256 per step), so after one binary search a cursor that
    // advances over the few tile starts in between finds each one.
    int cur = 0;
    {
      const uint32_t r = static_cast<uint32_t>(g_lo + tid);
      int hi = kGatherTiles;
#pragma unroll
      for (int step = 0; step < 8; ++step) {  // log2(kGatherTiles) halvings
        const int mid = (cur + hi) >> 1;
        if (rpref[mid] <= r) cur = mid; else hi = mid;
      }
    }
    for (uint64_t r0 = tid; r0 < g_total; r0 += kThreads * U) {
      uint64_t src[U], dst[U];
      uint32_t val[U], pos[U];
      bool live[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t r = static_cast<uint32_t>(g_lo + r0 + u * kThreads);
        while (cur + 1 < kGatherTiles && rpref[cur + 1] <= r) ++cur;
        const int lo = cur;
        const uint32_t in_tile = r - rpref[lo];
        dst[u] = tpref[lo] + in_tile;
        live[u] = r0 + u * kThreads < g_total && dst[u] < a.capacity;
        src[u] = (t0 + lo) * kTileCap<FMT> + in_tile;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!live[u]) continue;
        val[u] = __ldg(a.scr_val + src[u]);
        if constexpr (POSB == 1) pos[u] = __ldg(a.scr_pos + src[u]);
        else if constexpr (POSB == 2) pos[u] = __ldg(reinterpret_cast<const uint16_t*>(a.scr_pos) + src[u]);
        else if constexpr (POSB == 4) pos[u] = __ldg(reinterpret_cast<const uint32_t*>(a.scr_pos) + src[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!live[u]) continue;
        a.values[dst[u]] = static_cast<uint8_t>(val[u]);
        if constexpr (POSB == 1) a.positions[dst[u]] = static_cast<uint8_t>(pos[u]);
        else if constexpr (POSB == 2) reinterpret_cast<uint16_t*>(a.positions)[dst[u]] = static_cast<uint16_t>(pos[u]);
        else if constexpr (POSB == 4) reinterpret_cast<uint32_t*>(a.positions)[dst[u]] = pos[u];
      }
    }
  }
  // Escape-heavy tiles go to K2c (one CTA each, all of them in parallel).
  if (warp == 0 && part == 0) {
#pragma unroll
    for (int j = 0; j < kGatherTiles / 32; ++j) {
      const int k = j * 32 + lane;
      const uint64_t tile = t0 + k;
      if (tile < a.num_tiles && tcnt[k] > kTileCap<FMT>) {
        const unsigned int slot = atomicAdd(a.heavy_count, 1u);
        a.heavy_list[slot] = static_cast<uint32_t>(tile);
        a.heavy_pref[slot] = tpref[k];
      }
    }
  }
}

// ------------------------------------------------------------------ K2c
// Escape-heavy tiles (more escapes than a scratch slot holds): one CTA per
// listed tile re-derives its escapes from the input in element order.  Per
// round of 256 x 64 bytes: every thread loads its 64 bytes (all loads in
// flight) and parks them in shared memory, builds its escape mask from the
// marked LUT, one block scan gives each thread its first ordinal, threads
// append the tile-local indices of their escapes to a compact shared list,
// and then the whole CTA writes the round's records with consecutive threads
// on consecutive ordinals (coalesced stores, work spread evenly however the
// escapes cluster).  The grid is a fixed wave of CTAs striding over the list,
// so with no heavy tile the launch costs one load per CTA.
template <int FMT>
constexpr int kHeavySmem = kThreads * 64 + kThreads * (64 / Fmt<FMT>::kWordBytes) * 2;

template <int FMT, int POSB>
__global__ void __launch_bounds__(kThreads)
    escape_heavy(const __grid_constant__ sz_params p, const GatherArgs a) {
  constexpr int WB = Fmt<FMT>::kWordBytes;
  constexpr int EPT = 64 / WB;              // words per thread per round
  constexpr int RE = kThreads * EPT;        // elements per round
  // escape-flag lane tables: tf[k][e] = escape(e) << k, so the sum of a
  // 4-element group's lookups (lane k = element k) is its 4-bit flag nibble
  // (t4_group's addressing, flags only); 64 B / 128 B / 1 KiB per lane
  // for E4M3 / E5M2 / BF16
  constexpr int TB = 1 << Fmt<FMT>::kExpBits;
  __shared__ __align__(1024) uint32_t tf[4 * TB];
  __shared__ uint32_t hspine[kWarps];
  extern __shared__ __align__(16) uint8_t heavy_smem[];     // kHeavySmem<FMT> bytes
  uint32_t* const s_w = reinterpret_cast<uint32_t*>(heavy_smem);  // the round's words
  uint16_t* const s_idx = reinterpret_cast<uint16_t*>(heavy_smem + kThreads * 64);  // escapes
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_trigger();
  pdl_wait();
  const unsigned int count = *a.heavy_count;
  if (blockIdx.x >= count) return;
  for (int i = tid; i < 4 * TB; i += kThreads)
    tf[i] = static_cast<uint32_t>((p.enc_lut[i % TB] >> 4) & 1u) << (i / TB);
  __syncthreads();
  const uint32_t tbase = smem_addr(tf);
  // this thread's 64 bytes of round r0 (clipped at the tile end e_end)
  auto load_round = [&](uint64_t r0, uint64_t e_end, uint32_t (&w)[16]) {
    const uint64_t my0 = r0 + static_cast<uint64_t>(tid) * EPT;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two 32-byte halves (a segment holds >= 32 B)
      const uint64_t e = my0 + h * (32 / WB);
      const uint64_t off = e * WB;
      const uint8_t* src = a.words + off;
      if (a.seg_addrs)
        src = reinterpret_cast<const uint8_t*>(__ldg(a.seg_addrs + (off >> a.seg_shift))) +
              (off & ((1ull << a.seg_shift) - 1));
      if (e + 32 / WB <= e_end) {
        const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(src));
        const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
        w[8 * h + 0] = v0.x; w[8 * h + 1] = v0.y; w[8 * h + 2] = v0.z; w[8 * h + 3] = v0.w;
        w[8 * h + 4] = v1.x; w[8 * h + 5] = v1.y; w[8 * h + 6] = v1.z; w[8 * h + 7] = v1.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // clipped: whole words while inside
          uint32_t v = 0;
#pragma unroll
          for (int b = 0; b < 4 / WB; ++b) {
            const uint64_t j = q * (4 / WB) + b;
            if (e + j < e_end) {
              const uint32_t x = WB == 2 ? reinterpret_cast<const uint16_t*>(src)[j] : src[j];
              v |= x << (8 * WB * b);
            }
          }
          w[8 * h + q] = v;
        }
      }
    }
  };
  // Flat loop over (listed tile, round) with the next round's loads in
  // flight while this one is classified and written.
  unsigned int li = blockIdx.x;
  uint64_t e_begin = static_cast<uint64_t>(a.heavy_list[li]) * a.tile_elems;
  uint64_t e_end = min(e_begin + a.tile_elems, a.n);
  uint64_t ord = a.heavy_pref[li];
  uint64_t r0 = e_begin;
  uint32_t w[16];
  load_round(r0, e_end, w);
  while (true) {
    // the round after this one
    unsigned int nli = li;
    uint64_t nr0 = r0 + RE, ne_end = e_end, nbegin = e_begin;
    if (nr0 >= e_end) {
      nli = li + gridDim.x;
      if (nli < count) {
        nbegin = static_cast<uint64_t>(a.heavy_list[nli]) * a.tile_elems;
        ne_end = min(nbegin + a.tile_elems, a.n);
        nr0 = nbegin;
      }
    }
    uint32_t wn[16];
    if (nli < count) load_round(nr0, ne_end, wn);
    {
      const uint64_t my0 = r0 + static_cast<uint64_t>(tid) * EPT;
      // 16-byte chunk c of thread t at chunk c ^ ((t >> 1) & 3): each 8-lane
      // store phase then covers all 32 banks (linear: 4-way conflicts)
      const uint32_t csw = (tid >> 1) & 3;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(&s_w[tid * 16 + 4 * (q ^ csw)]) =
            make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      // elements of this thread inside the tile
      const uint32_t nvalid =
          e_end > my0 ? static_cast<uint32_t>(min(e_end - my0, static_cast<uint64_t>(EPT))) : 0u;
      uint32_t mask[EPT / 32];
      uint32_t cnt = 0;
#pragma unroll
      for (int q = 0; q < EPT / 32; ++q) {
        uint32_t mk = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {  // group of 4 elements -> flag nibble g
          uint32_t t0, t1, t2, t3;
          if constexpr (WB == 2) {
            const uint32_t f0 = (w[2 * g] >> 5) & 0x03FC03FCu;  // 4e of elements 4g, 4g+1
            const uint32_t f1 = (w[2 * g + 1] >> 5) & 0x03FC03FCu;
            t0 = lds_u32_off<0>(tbase + (f0 & 0xFFFFu));
            t1 = lds_u32_off<4 * TB>(tbase + (f0 >> 16));
            t2 = lds_u32_off<8 * TB>(tbase + (f1 & 0xFFFFu));
            t3 = lds_u32_off<12 * TB>(tbase + (f1 >> 16));
          } else {
            const uint32_t x = w[8 * q + g];
            const uint32_t f = FMT == SZ_E5M2 ? (x & 0x7C7C7C7Cu)           // byte k = 4e
                                              : ((x >> 1) & 0x3C3C3C3Cu);
            t0 = lds_u32_off<0>(__byte_perm(f, tbase, 0x7650));
            t1 = lds_u32_off<4 * TB>(__byte_perm(f, tbase, 0x7651));
            t2 = lds_u32_off<8 * TB>(__byte_perm(f, tbase, 0x7652));
            t3 = lds_u32_off<12 * TB>(__byte_perm(f, tbase, 0x7653));
          }
          mk |= (t0 + t1 + t2 + t3) << (4 * g);
        }
        const uint32_t nv = nvalid > 32u * q ? nvalid - 32u * q : 0u;
        if (nv < 32) mk &= (1u << nv) - 1u;
        mask[q] = mk;
        cnt += __popc(mk);
      }
      // block exclusive scan of cnt
      uint32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
      }
      if (lane == 31) hspine[warp] = incl;
      __syncthreads();
      uint32_t wbase = 0, total = 0;
#pragma unroll
      for (int v = 0; v < kWarps; ++v) {
        const uint32_t t = hspine[v];
        wbase += v < warp ? t : 0;
        total += t;
      }
      uint32_t r = wbase + incl - cnt;  // this thread's first round-relative ordinal
#pragma unroll
      for (int q = 0; q < EPT / 32; ++q) {
        uint32_t mk = mask[q];
        while (mk) {
          const int j = __ffs(mk) - 1;
          mk &= mk - 1;
          s_idx[r++] = static_cast<uint16_t>(tid * EPT + q * 32 + j);
        }
      }
      __syncthreads();
      // (explicit shared-space loads: the extern-smem pointers reach here as
      // generic addresses)
      const uint32_t w_sa = smem_addr(s_w), i_sa = smem_addr(s_idx);
      for (uint32_t k = tid; k < total; k += kThreads) {
        const uint64_t o = ord + k;
        if (o < a.capacity) {
          const uint32_t el = lds_u16(i_sa + 2 * k);
          const uint32_t b = el * WB;  // byte of the round: thread b >> 6, chunk (b >> 4) & 3
          const uint32_t phys = (b & ~0x30u) | ((((b >> 4) ^ (b >> 7)) & 3u) << 4);
          const uint32_t word = WB == 2 ? lds_u16(w_sa + phys) : lds_u8(w_sa + phys);
          a.values[o] = static_cast<uint8_t>(raw_exponent<FMT>(word));
          put_position<POSB>(a.positions, o, r0 + el, a.chunk, a.chunk_shift);
        }
      }
      ord += total;
      __syncthreads();  // s_w / s_idx / hspine reuse
    }
    if (nli >= count) break;
    if (nli != li) ord = a.heavy_pref[nli];
    li = nli;
    r0 = nr0;
    e_end = ne_end;
    e_begin = nbegin;
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = wn[i];
  }
}

// K6: raw exponent bytes -> dense LE bitstream of W bits per value
// (_pack_values / _pack_bits, codec.py:241-266; formats.py:167-189), FP8
// escape values at W = 5 / 4.  Reads M from device memory so it chains
// after the encoder without a host round trip.
// One thread per 32 values: 32 W-bit values are exactly W 32-bit
// words of the LE stream, so a thread loads its 32 bytes (two 16-byte loads,
// both in flight), places every value at a compile-time bit offset, and
// stores its W words straight to global memory (a warp's stores cover one
// contiguous 128 x W-byte run).  Unaligned pointers and the ragged end take
// byte loads / stores.
template <int W>
__global__ void __launch_bounds__(kThreads)
    pack_values32_kernel(const uint8_t* __restrict__ vals, const uint64_t* m_ptr,
                         uint64_t capacity, uint8_t* __restrict__ out) {
  const uint64_t m = min(*m_ptr, capacity);
  const uint64_t units = (m + 31) / 32;
  const uint64_t nbytes_total = (m * W + 7) / 8;
  const bool v16 = !(reinterpret_cast<uintptr_t>(vals) & 15);
  const bool o4 = !(reinterpret_cast<uintptr_t>(out) & 3);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < units;
       u += stride) {
    uint32_t x[8];
    const bool full = u * 32 + 32 <= m;
    if (v16 && full) {
      const uint4* src = reinterpret_cast<const uint4*>(vals) + 2 * u;
      const uint4 a = __ldg(src), b = __ldg(src + 1);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
      x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = 0;
      for (int j = 0; j < 32; ++j)
        if (u * 32 + j < m) x[j >> 2] |= static_cast<uint32_t>(vals[u * 32 + j]) << (8 * (j & 3));
    }
    uint32_t w[W];
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t v = (x[j >> 2] >> (8 * (j & 3))) & ((1u << W) - 1u);
      const int bit = j * W, k = bit >> 5, off = bit & 31;
      w[k] |= v << off;
      if (off + W > 32) w[k + 1] |= v >> (32 - off);
    }
    const uint64_t ob = u * 4 * W;
    if (o4 && ob + 4 * W <= nbytes_total) {
      uint32_t* d = reinterpret_cast<uint32_t*>(out + ob);
#pragma unroll
      for (int k = 0; k < W; ++k) d[k] = w[k];
    } else {
      for (int b = 0; b < 4 * W; ++b)
        if (ob + b < nbytes_total) out[ob + b] = static_cast<uint8_t>(w[b >> 2] >> (8 * (b & 3)));
    }
  }
}

}  // namespace sz

// ============================================================ host dispatch
namespace {

using namespace sz;

uint64_t encode_tile_for(uint32_t fmt) {
  return static_cast<uint64_t>(kEncSlots) * (fmt == SZ_BF16 ? 16 : 32);
}
uint64_t tile_cap_for(uint32_t fmt) {
  return fmt == SZ_BF16 ? kTileCap<SZ_BF16> : (fmt == SZ_E5M2 ? kTileCap<SZ_E5M2> : kTileCap<SZ_E4M3>);
}
int pos_bytes(const sz_params* p) {
  return p->sentinel ? 0 : (p->abs32 ? 4 : (p->chunk_size <= 256 ? 1 : 2));
}

// Workspace layout (all offsets 256-byte aligned):
//   [tile counter | gather counter | gather look-back states]  -> zeroed per call
//   tile_esc[num_tiles] u32, scratch positions, scratch values
struct EncWs {
  unsigned long long* tile_counter;
  unsigned long long* gather_counter;
  uint64_t* snapshot;
  uint64_t* states;          // tile-prefix scan look-back states
  unsigned long long* scan_counter;
  uint64_t* tile_pref;
  uint32_t* tile_esc;
  uint8_t* scr_pos;
  uint8_t* scr_val;
  unsigned int* heavy_count;
  uint32_t* heavy_list;
  uint64_t* heavy_pref;
  size_t zero_bytes;
  size_t total;
};

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

EncWs carve(void* base, uint64_t n, const sz_params* p) {
  EncWs w{};
  const uint64_t tiles = (n + encode_tile_for(p->fmt) - 1) / encode_tile_for(p->fmt);
  const int pb = pos_bytes(p) ? pos_bytes(p) : 1;
  uint8_t* b = static_cast<uint8_t*>(base);
  size_t off = 0;
  w.tile_counter = reinterpret_cast<unsigned long long*>(b + off);
  w.gather_counter = w.tile_counter + 1;
  w.snapshot = reinterpret_cast<uint64_t*>(w.tile_counter + 2);
  w.heavy_count = reinterpret_cast<unsigned int*>(w.tile_counter + 3);
  w.scan_counter = w.tile_counter + 4;
  w.states = reinterpret_cast<uint64_t*>(w.tile_counter + 5);
  off = align256((5 + offsets_tiles(tiles)) * sizeof(uint64_t));
  w.zero_bytes = off;
  w.tile_esc = reinterpret_cast<uint32_t*>(b + off);
  off = align256(off + tiles * sizeof(uint32_t));
  const uint64_t cap = tile_cap_for(p->fmt);
  w.scr_pos = b + off;
  off = align256(off + tiles * cap * pb);
  w.scr_val = b + off;
  off = align256(off + tiles * cap);
  w.heavy_list = reinterpret_cast<uint32_t*>(b + off);
  off = align256(off + tiles * sizeof(uint32_t));
  w.heavy_pref = reinterpret_cast<uint64_t*>(b + off);
  off = align256(off + tiles * sizeof(uint64_t));
  w.tile_pref = reinterpret_cast<uint64_t*>(b + off);
  off = align256(off + (tiles + 1) * sizeof(uint64_t));
  w.total = off;
  return w;
}


template <int FMT, int CB, int POSB>
cudaError_t launch_encode(const sz_params& p, const EncodeArgs& a, const GatherArgs& g,
                          const CUtensorMap& tm, cudaStream_t s) {
  auto kern = encode_tiles<FMT, CB, POSB>;
  const int smem = static_cast<int>(sizeof(EncSmem<FMT, CB>)) + 1024;  // + alignment slack
  const KernelSetup ks = kernel_setup(reinterpret_cast<const void*>(kern), smem, kEncThreads<FMT, CB>);
  if (ks.err != cudaSuccess) return ks.err;
  cudaError_t e;
  const uint64_t want = static_cast<uint64_t>(ks.sms);
  const unsigned grid = static_cast<unsigned>(a.num_tiles < want ? a.num_tiles : want);
  e = launch_pdl(kern, dim3(grid), dim3(kEncThreads<FMT, CB>), smem, s, p, a, tm);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  {
    OffsetsArgs oa{};
    oa.counts = a.tile_esc;
    oa.n_counts = a.num_tiles;
    oa.offsets = const_cast<uint64_t*>(g.tile_pref);
    oa.states = g.scan_states;
    oa.tile_counter = g.scan_counter;
    oa.num_tiles = offsets_tiles(a.num_tiles);
    e = launch_pdl(offsets_kernel, dim3(static_cast<unsigned>(oa.num_tiles)), dim3(kThreads), 0,
                   s, oa);
    if (e != cudaSuccess) return e;
  }
  e = launch_pdl(escape_gather<FMT, POSB>, dim3(static_cast<unsigned>(g.num_groups * g.split)),
                 dim3(kThreads), 0, s, p, g);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // one wave of K2c CTAs (as many as fit per SM next to nothing else)
  const KernelSetup hs = kernel_setup(reinterpret_cast<const void*>(escape_heavy<FMT, POSB>),
                                      kHeavySmem<FMT>, kThreads);
  const int heavy_per_sm = hs.err == cudaSuccess ? hs.per_sm : 0;
  if (heavy_per_sm <= 0) return cudaErrorInvalidConfiguration;
  const uint64_t heavy_grid = want * static_cast<uint64_t>(heavy_per_sm);
  return launch_pdl(escape_heavy<FMT, POSB>,
                    dim3(static_cast<unsigned>(heavy_grid < a.num_tiles ? heavy_grid : a.num_tiles)),
                    dim3(kThreads), kHeavySmem<FMT>, s, p, g);
}

template <int FMT, int CB>
cudaError_t dispatch_pos(int posb, const sz_params& p, const EncodeArgs& a, const GatherArgs& g,
                         const CUtensorMap& tm, cudaStream_t s) {
  switch (posb) {
    case 0: return launch_encode<FMT, CB, 0>(p, a, g, tm, s);
    case 1: return launch_encode<FMT, CB, 1>(p, a, g, tm, s);
    case 2: return launch_encode<FMT, CB, 2>(p, a, g, tm, s);
    default: return launch_encode<FMT, CB, 4>(p, a, g, tm, s);
  }
}

template <int FMT>
cudaError_t dispatch_cb(int posb, const sz_params& p, const EncodeArgs& a, const GatherArgs& g,
                        const CUtensorMap& tm,
                        cudaStream_t s) {
  return p.code_bits == 4 ? dispatch_pos<FMT, 4>(posb, p, a, g, tm, s)
                          : dispatch_pos<FMT, 3>(posb, p, a, g, tm, s);
}

// Input words as a 2-D byte tensor [rows][128] (full 128-byte rows only),
// boxes of 256 rows = one 32 KiB encoder tile, 128B swizzle.  Returns false
// (caller falls back to 1-D bulk copies) when the driver entry point is
// unavailable or the input has no full tile.
bool make_input_tmap(const void* words, uint64_t n_bytes, CUtensorMap* tm,
                     uint32_t box_rows = kEncTileBytes / 128) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode_fn = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode_fn || n_bytes < static_cast<uint64_t>(box_rows) * 128) return false;
  const cuuint64_t dims[2] = {128, n_bytes / 128};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode_fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(words), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

extern "C" {

int sz_record_cuda(cudaError_t e);  // sz_misc.cu
int sz_check_params(const sz_params* p, int decode_side);

size_t sz_encode_workspace_bytes(uint64_t n, const sz_params* p) {
  if (!p || p->fmt > SZ_E4M3) return 0;
  return carve(nullptr, n, p).total + 256;
}

}  // extern "C"

namespace {
// Shared body of sz_encode (contiguous words) and sz_encode_segments (paged:
// d_words null, segment table + log2 segment bytes).
int encode_impl(const void* d_words, const uint64_t* seg_addrs, uint32_t seg_shift, uint64_t n,
                const sz_params* p, const sz_encoded* out, void* d_ws, size_t ws_bytes,
                void* stream, uint64_t va_lo = 0, uint64_t va_hi = 0) {
  if (int rc = sz_check_params(p, 0)) return rc;
  if (n == 0 || !out || (!d_words && !seg_addrs)) return SZ_ECONFIG;
  if ((reinterpret_cast<uintptr_t>(d_words) & 31) ||
      (reinterpret_cast<uintptr_t>(out->d_codes) & 15) ||
      (reinterpret_cast<uintptr_t>(out->d_sm) & 15) || (reinterpret_cast<uintptr_t>(d_ws) & 255))
    return SZ_EALIGN;
  if (ws_bytes < sz_encode_workspace_bytes(n, p)) return SZ_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int exp_bits = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 5 : 4);
  const int sm_bits = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 3 : 4);
  const bool chunked = !p->sentinel && !p->abs32;
  const int epv = p->fmt == SZ_BF16 ? 16 : 32;
  const uint64_t tile = encode_tile_for(p->fmt);
  const EncWs w = carve(d_ws, n, p);

  EncodeArgs a{};
  a.words = static_cast<const uint8_t*>(d_words);
  a.seg_addrs = seg_addrs;
  a.seg_shift = seg_shift;
  a.n = n;
  a.codes = static_cast<uint8_t*>(out->d_codes);
  a.sm = static_cast<uint8_t*>(out->d_sm);
  a.counts = out->d_counts;
  a.num_tiles = (n + tile - 1) / tile;
  a.n_chunks = chunked ? (n + p->chunk_size - 1) / p->chunk_size : 0;
  a.codes_len = (n * p->code_bits + 7) / 8;
  a.sm_len = (n * sm_bits + 7) / 8;
  a.chunk = p->chunk_size;
  a.chunk_shift = (p->chunk_size & (p->chunk_size - 1)) == 0 ? __builtin_ctz(p->chunk_size) : -1;
  a.counts_mode = 0;
  a.lut_stride = 4;
  a.one = 1;
  a.k_lo = 1057u << 10;
  a.k_hi = 1057u;
  a.tile_counter = w.tile_counter;
  a.tile_esc = w.tile_esc;
  a.scr_pos = w.scr_pos;
  a.scr_val = w.scr_val;
  a.escape_base = out->d_escape_base;
  a.base_snapshot = w.snapshot;
  if (chunked) {
    if (!out->d_counts) return SZ_ECONFIG;
    a.counts_mode = (tile % p->chunk_size == 0 && p->chunk_size % epv == 0) ? 1 : 2;
  }
  if (out->escape_capacity && (!out->d_values || (!p->sentinel && !out->d_positions)))
    return SZ_ECONFIG;

  GatherArgs g{};
  g.words = a.words;
  g.seg_addrs = seg_addrs;
  g.seg_shift = seg_shift;
  g.n = n;
  g.tile_esc = w.tile_esc;
  g.scr_pos = w.scr_pos;
  g.scr_val = w.scr_val;
  g.num_tiles = a.num_tiles;
  g.tile_elems = tile;
  g.positions = static_cast<uint8_t*>(out->d_positions);
  g.values = out->d_values;
  g.capacity = out->escape_capacity;
  g.n_escapes = out->d_n_escapes;
  g.tile_pref = w.tile_pref;
  g.scan_states = w.states;
  g.scan_counter = w.scan_counter;
  g.counter = w.gather_counter;
  g.num_groups = (a.num_tiles + kGatherTiles - 1) / kGatherTiles;
  g.chunk = a.chunk;
  g.chunk_shift = a.chunk_shift;
  g.base_snapshot = w.snapshot;
  g.escape_base = out->d_escape_base;
  g.heavy_list = w.heavy_list;
  // CTAs per group: >= ~2048 record movers in all, so escape-dense inputs
  // (~1100 records per tile) keep enough loads in flight; sparse groups cost
  // each extra CTA one 1 KiB tile-count load and an early exit
  {
    const uint64_t want = (2048 + g.num_groups - 1) / g.num_groups;
    g.split = static_cast<uint32_t>(want < 1 ? 1 : (want > 64 ? 64 : want));
  }
  g.heavy_pref = w.heavy_pref;
  g.heavy_count = w.heavy_count;

  cudaError_t e = cudaMemsetAsync(d_ws, 0, w.zero_bytes, s);
  if (e == cudaSuccess && a.counts_mode == 2)
    e = cudaMemsetAsync(out->d_counts, 0, a.n_chunks * sizeof(uint32_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);

#ifdef SZ_TIMERS
  static const bool dbg_timers = std::getenv("SZ_DEBUG_TIMERS") != nullptr;
#else
  constexpr bool dbg_timers = false;  // build with -DSZ_TIMERS for role timers
#endif
  unsigned long long* dbg = nullptr;
  if (dbg_timers) {
    cudaMalloc(&dbg, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), s);
    a.dbg = dbg;
  }
  alignas(64) CUtensorMap tm{};
  if (!seg_addrs) {
    a.use_tmap = make_input_tmap(d_words, n * (p->fmt == SZ_BF16 ? 2 : 1), &tm);
  } else if (va_hi > va_lo && !(va_lo & 127) && seg_shift >= 10 &&
             (va_hi - va_lo) / 128 < (1ull << 31)) {
    // segments of >= 1 KiB (whole 8-row swizzle atoms) inside a window whose
    // rows fit the int32 box coordinate
    const uint64_t seg = 1ull << seg_shift;
    const uint32_t rows = static_cast<uint32_t>(
        (seg < static_cast<uint64_t>(kEncTileBytes) ? seg : kEncTileBytes) / 128);
    a.seg_tmap = make_input_tmap(reinterpret_cast<const void*>(va_lo),
                                 (va_hi - va_lo + 127) & ~127ull, &tm, rows);
    a.use_tmap = a.seg_tmap;
    a.seg_va_lo = va_lo;
  }
  const int posb = pos_bytes(p);
  switch (p->fmt) {
    case SZ_BF16: e = dispatch_cb<SZ_BF16>(posb, *p, a, g, tm, s); break;
    case SZ_E5M2: e = dispatch_cb<SZ_E5M2>(posb, *p, a, g, tm, s); break;
    default: e = dispatch_cb<SZ_E4M3>(posb, *p, a, g, tm, s); break;
  }
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (dbg) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr,
                 "[sz_encode timers] dense wait=%llu work=%llu | writer wait=%llu work=%llu"
                 " | producer in_empty=%llu scan_empty=%llu\n",
                 h[0], h[1], h[2], h[3], h[6], h[7]);
    cudaFree(dbg);
  }
  // (append mode: the caller packs the whole stream once, after the last piece)
  if (exp_bits != 8 && out->escape_capacity && !out->d_escape_base) {
    if (!out->d_values_packed) return SZ_ECONFIG;
    // one thread per 32 values of the capacity (threads past M exit at
    // once), at most 8 blocks per SM with a grid-stride loop beyond
    const uint64_t want = (out->escape_capacity + 32 * kThreads - 1) / (32 * kThreads);
    const unsigned pg = static_cast<unsigned>(want < 148 * 8 ? (want ? want : 1) : 148 * 8);
    if (exp_bits == 5)
      pack_values32_kernel<5><<<pg, kThreads, 0, s>>>(out->d_values, out->d_n_escapes,
                                                      out->escape_capacity, out->d_values_packed);
    else
      pack_values32_kernel<4><<<pg, kThreads, 0, s>>>(out->d_values, out->d_n_escapes,
                                                      out->escape_capacity, out->d_values_packed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return sz_record_cuda(e);
  }
  return SZ_OK;
}
}  // namespace

extern "C" {

int sz_encode(const void* d_words, uint64_t n, const sz_params* p, const sz_encoded* out,
              void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_words) return SZ_ECONFIG;
  return encode_impl(d_words, nullptr, 0, n, p, out, d_ws, ws_bytes, stream);
}

int sz_encode_segments(const uint64_t* d_seg_addrs, uint64_t n_segs, uint64_t seg_bytes,
                       const sz_params* p, const sz_encoded* out, void* d_ws, size_t ws_bytes,
                       void* stream) {
  return sz_encode_segments_va(d_seg_addrs, n_segs, seg_bytes, 0, 0, p, out, d_ws, ws_bytes,
                               stream);
}

int sz_encode_segments_va(const uint64_t* d_seg_addrs, uint64_t n_segs, uint64_t seg_bytes,
                          uint64_t va_lo, uint64_t va_hi, const sz_params* p,
                          const sz_encoded* out, void* d_ws, size_t ws_bytes, void* stream) {
  if (!p || !d_seg_addrs || n_segs == 0 || seg_bytes < 32 || (seg_bytes & (seg_bytes - 1)))
    return SZ_ECONFIG;
  const uint64_t wb = p->fmt == SZ_BF16 ? 2 : 1;
  return encode_impl(nullptr, d_seg_addrs, static_cast<uint32_t>(__builtin_ctzll(seg_bytes)),
                     n_segs * seg_bytes / wb, p, out, d_ws, ws_bytes, stream, va_lo, va_hi);
}

}  // extern "C"
