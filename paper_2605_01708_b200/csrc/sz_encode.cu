// sz_encode.cu — K2: single-pass SplitZip encoder for sm_100a.
//
// Replaces codec.py:299-321 (encode) and its byte-identical Quad64 variant
// codec.py:324-401 (encode_quad).  One CTA = one tile of
// ITEMS x 256 x EPV elements (EPV = 16 BF16 / 32 FP8 words = one 32-byte
// vector per "slot"; slot s = item * 256 + thread, element order).
//
//   1. 256-bit streaming loads of the tile (LDG.E.256, L1 no-allocate).
//   2. Per 4 elements: split fields with byte permutes, look the exponents up
//      in the marked LUT (shared memory; bit 4 = escape, low bits = code to
//      store, as in encode_quad's marked table codec.py:340-342), pack the
//      codes (4-bit nibbles or 3-bit LE stream) and the sign|mantissa plane
//      (byte plane for BF16, 3/4-bit LE stream for FP8), store both with
//      vector stores.  Escape flags come out of the same LUT byte.
//   3. Escape compaction in ascending element order: per-slot popc counts,
//      block-wide exclusive scan in slot order, decoupled look-back across
//      tiles (dynamic tile ids => forward progress), then each thread writes
//      its escapes' (position, raw exponent) records at their global ordinal.
//   4. Per-chunk escape counts (codec.py:292-295): directly from the block
//      scan when chunks tile the CTA tile, else by integer atomics into a
//      zeroed array (deterministic: the sums do not depend on order).
#include "sz_common.cuh"

namespace sz {

struct EncodeArgs {
  const uint8_t* words;
  uint64_t n;
  uint8_t* codes;
  uint8_t* sm;
  uint32_t* counts;
  void* positions;
  uint8_t* values;
  uint64_t* n_escapes;
  uint64_t capacity;
  uint64_t* states;
  unsigned long long* tile_counter;
  uint64_t num_tiles;
  uint64_t n_chunks;
  uint64_t codes_len;
  uint64_t sm_len;
  uint32_t chunk;
  int32_t chunk_shift;   // log2(chunk) when a power of two, else -1
  int32_t counts_mode;   // 0 none, 1 direct from scan, 2 atomics (pre-zeroed)
};

template <int FMT>
__device__ __forceinline__ void split_group(const uint32_t (&x)[8], int g, uint32_t& e4,
                                            uint32_t& a4) {
  if constexpr (FMT == SZ_BF16) {
    // Elements 4g..4g+3 live in words 2g, 2g+1 (two little-endian u16 each).
    const uint32_t lo4 = __byte_perm(x[2 * g], x[2 * g + 1], 0x6420);
    const uint32_t hi4 = __byte_perm(x[2 * g], x[2 * g + 1], 0x7531);
    e4 = ((hi4 << 1) & 0xFEFEFEFEu) | ((lo4 >> 7) & 0x01010101u);
    a4 = (hi4 & 0x80808080u) | (lo4 & 0x7F7F7F7Fu);
  } else if constexpr (FMT == SZ_E5M2) {
    e4 = (x[g] >> 2) & 0x1F1F1F1Fu;
    a4 = ((x[g] >> 5) & 0x04040404u) | (x[g] & 0x03030303u);
  } else {
    e4 = (x[g] >> 3) & 0x0F0F0F0Fu;
    a4 = ((x[g] >> 4) & 0x08080808u) | (x[g] & 0x07070707u);
  }
}

__device__ __forceinline__ uint32_t lut4(const uint8_t* lut, uint32_t e4) {
  const uint32_t m0 = lut[e4 & 0xFF], m1 = lut[(e4 >> 8) & 0xFF];
  const uint32_t m2 = lut[(e4 >> 16) & 0xFF], m3 = lut[e4 >> 24];
  return __byte_perm(__byte_perm(m0, m1, 0x0040), __byte_perm(m2, m3, 0x0040), 0x5410);
}

template <int FMT, int CB, int POSB, int ITEMS>
__global__ void __launch_bounds__(kThreads)
    encode_kernel(const __grid_constant__ sz_params p, const EncodeArgs a) {
  constexpr int EPV = kEpv<FMT>;
  constexpr int G = EPV / 4;
  constexpr int WB = Fmt<FMT>::kWordBytes;
  constexpr int SMB = Fmt<FMT>::kSmBits;
  constexpr int CBYTES = EPV * CB / 8;
  constexpr int SBYTES = EPV * SMB / 8;
  constexpr int CWORDS = (CBYTES + 3) / 4;
  constexpr int SWORDS = (SBYTES + 3) / 4;
  constexpr int SLOTS = ITEMS * kThreads;
  constexpr uint64_t TILE = static_cast<uint64_t>(SLOTS) * EPV;

  __shared__ uint8_t lut[256];
  __shared__ BlockScanSmem<ITEMS> scan_sm;
  __shared__ uint32_t s_prefix[SLOTS + 1];
  __shared__ unsigned long long s_tile;
  __shared__ uint64_t s_excl;

  const int tid = threadIdx.x;
  for (int i = tid; i < 256; i += kThreads) lut[i] = p.enc_lut[i];
  if (tid == 0) s_tile = atomicAdd(a.tile_counter, 1ull);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tile_e0 = tile * TILE;
  const uint64_t n = a.n;

  // ---- 1. loads (all items in flight before any compute)
  uint32_t x[ITEMS][8];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t e0 = tile_e0 + static_cast<uint64_t>(i * kThreads + tid) * EPV;
    if (e0 + EPV <= n) {
      ld_stream256(a.words + e0 * WB, x[i]);
    } else {
      ld_bytes_clipped<32>(a.words, e0 * WB, x[i], e0 < n ? n * WB : 0);
    }
  }

  // ---- 2. dense transform + stores
  uint32_t fmask[ITEMS];
  uint32_t cnt[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t e0 = tile_e0 + static_cast<uint64_t>(i * kThreads + tid) * EPV;
    const bool full = e0 + EPV <= n;
    const int nv = full ? EPV : (e0 < n ? static_cast<int>(n - e0) : 0);
    uint32_t mk[G], ag[G];
    uint32_t any = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t e4, a4;
      split_group<FMT>(x[i], g, e4, a4);
      uint32_t m4 = lut4(lut, e4);
      if (!full) {
        const int v = min(max(nv - 4 * g, 0), 4);
        const uint32_t keep = v >= 4 ? 0xFFFFFFFFu : ((1u << (8 * v)) - 1u);
        m4 &= keep;
        a4 &= keep;
      }
      mk[g] = m4;
      ag[g] = a4;
      any |= m4;
    }
    uint32_t fm = 0;
    if (any & 0x10101010u) {
#pragma unroll
      for (int g = 0; g < G; ++g) fm |= flags4(mk[g]) << (4 * g);
    }
    fmask[i] = fm;
    cnt[i] = __popc(fm);

    uint32_t cw[CWORDS], sw[SWORDS];
    {
      uint32_t grp[G];
      if constexpr (CB == 4) {
#pragma unroll
        for (int g = 0; g < G; ++g) grp[g] = pack_nib4(mk[g] & 0x0F0F0F0Fu);
        concat_groups<G, 16>(grp, cw);
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g) grp[g] = pack_tri4(mk[g] & 0x07070707u);
        concat_groups<G, 12>(grp, cw);
      }
    }
    if constexpr (SMB == 8) {
#pragma unroll
      for (int g = 0; g < G; ++g) sw[g] = ag[g];
    } else {
      uint32_t grp[G];
      if constexpr (SMB == 4) {
#pragma unroll
        for (int g = 0; g < G; ++g) grp[g] = pack_nib4(ag[g]);
        concat_groups<G, 16>(grp, sw);
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g) grp[g] = pack_tri4(ag[g]);
        concat_groups<G, 12>(grp, sw);
      }
    }
    const uint64_t coff = e0 * CB / 8, soff = e0 * SMB / 8;
    if (full) {
      st_packed<CBYTES>(a.codes + coff, cw);
      st_packed<SBYTES>(a.sm + soff, sw);
    } else if (nv > 0) {
      st_bytes_clipped<CBYTES>(a.codes, coff, cw, a.codes_len);
      st_bytes_clipped<SBYTES>(a.sm, soff, sw, a.sm_len);
    }
  }

  // ---- 3. escape compaction: block scan + decoupled look-back
  uint32_t excl[ITEMS];
  const uint32_t total = block_scan<ITEMS>(cnt, excl, scan_sm);
  if (tid < 32) {
    const uint64_t ex = lookback_warp(a.states, tile, total);
    if (tid == 0) {
      s_excl = ex;
      if (tile == a.num_tiles - 1) *a.n_escapes = ex + total;
    }
  }
  if (a.counts_mode == 1) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) s_prefix[i * kThreads + tid + 1] = excl[i] + cnt[i];
    if (tid == 0) s_prefix[0] = 0;
  }
  __syncthreads();
  const uint64_t tile_excl = s_excl;

  bool per_escape_atomics = false;
  if (a.counts_mode == 2) {
    const uint64_t last = min(tile_e0 + TILE, n) - 1;
    const uint64_t k0 = tile_e0 / a.chunk, k1 = last / a.chunk;
    if (k0 == k1) {
      if (tid == 0 && total) atomicAdd(&a.counts[k0], total);
    } else {
      per_escape_atomics = true;
    }
  }

#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    uint32_t fm = fmask[i];
    if (!fm) continue;
    const uint64_t e0 = tile_e0 + static_cast<uint64_t>(i * kThreads + tid) * EPV;
    uint64_t ord = tile_excl + excl[i];
    while (fm) {
      const int j = __ffs(fm) - 1;
      fm &= fm - 1;
      const uint64_t idx = e0 + j;
      // Raw exponent: re-read the (L2-resident) word; escapes are rare, so
      // this is cheaper than holding the exponent bytes in registers.
      uint32_t ev;
      if constexpr (FMT == SZ_BF16) ev = (reinterpret_cast<const uint16_t*>(a.words)[idx] >> 7) & 0xFF;
      else if constexpr (FMT == SZ_E5M2) ev = (a.words[idx] >> 2) & 0x1F;
      else ev = (a.words[idx] >> 3) & 0x0F;
      if (ord < a.capacity) {
        a.values[ord] = static_cast<uint8_t>(ev);
        if constexpr (POSB == 4) {
          static_cast<uint32_t*>(a.positions)[ord] = static_cast<uint32_t>(idx);
        } else if constexpr (POSB == 2 || POSB == 1) {
          const uint64_t pos = a.chunk_shift >= 0 ? (idx & (a.chunk - 1)) : (idx % a.chunk);
          if constexpr (POSB == 2)
            static_cast<uint16_t*>(a.positions)[ord] = static_cast<uint16_t>(pos);
          else
            static_cast<uint8_t*>(a.positions)[ord] = static_cast<uint8_t>(pos);
        }
      }
      if (per_escape_atomics) atomicAdd(&a.counts[idx / a.chunk], 1u);
      ++ord;
    }
  }

  // ---- 4. per-chunk counts straight from the scan (chunks tile the CTA tile)
  if (a.counts_mode == 1) {
    const uint32_t slots_per_chunk = a.chunk / EPV;
    const uint32_t chunks_here = static_cast<uint32_t>(TILE / a.chunk);
    const uint64_t k_base = tile_e0 / a.chunk;
    for (uint32_t k = tid; k < chunks_here; k += kThreads) {
      if (k_base + k >= a.n_chunks) break;
      a.counts[k_base + k] = s_prefix[(k + 1) * slots_per_chunk] - s_prefix[k * slots_per_chunk];
    }
  }
}

// K6: raw exponent bytes -> dense LE bitstream of `width` bits per value
// (_pack_values / _pack_bits, codec.py:241-266).  Reads M from device memory
// so it chains after the encoder without a host round trip.
__global__ void pack_values_kernel(const uint8_t* __restrict__ vals, const uint64_t* m_ptr,
                                   uint64_t capacity, int width, uint8_t* __restrict__ out) {
  const uint64_t m = min(*m_ptr, capacity);
  const uint64_t groups = (m + 7) / 8;
  for (uint64_t gi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; gi < groups;
       gi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t acc = 0;
    for (int j = 0; j < 8; ++j) {
      const uint64_t o = gi * 8 + j;
      const uint64_t v = o < m ? vals[o] : 0;
      acc |= v << (j * width);
    }
    const uint64_t nbytes_total = (m * width + 7) / 8;
    for (int b = 0; b < width; ++b) {
      const uint64_t ob = gi * width + b;
      if (ob < nbytes_total) out[ob] = static_cast<uint8_t>(acc >> (8 * b));
    }
  }
}

}  // namespace sz

// ============================================================ host dispatch
namespace {

using namespace sz;

constexpr int kEncodeItems = 2;

template <int FMT>
constexpr uint64_t encode_tile() {
  return static_cast<uint64_t>(kEncodeItems) * kThreads * kEpv<FMT>;
}

uint64_t encode_tile_for(uint32_t fmt) {
  return fmt == SZ_BF16 ? encode_tile<SZ_BF16>() : encode_tile<SZ_E5M2>();
}

template <int FMT, int CB, int POSB>
void launch_encode(const sz_params& p, const EncodeArgs& a, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.num_tiles);
  encode_kernel<FMT, CB, POSB, kEncodeItems><<<grid, kThreads, 0, s>>>(p, a);
}

template <int FMT, int CB>
void dispatch_pos(int posb, const sz_params& p, const EncodeArgs& a, cudaStream_t s) {
  switch (posb) {
    case 0: launch_encode<FMT, CB, 0>(p, a, s); break;
    case 1: launch_encode<FMT, CB, 1>(p, a, s); break;
    case 2: launch_encode<FMT, CB, 2>(p, a, s); break;
    default: launch_encode<FMT, CB, 4>(p, a, s); break;
  }
}

template <int FMT>
void dispatch_cb(int posb, const sz_params& p, const EncodeArgs& a, cudaStream_t s) {
  if (p.code_bits == 4)
    dispatch_pos<FMT, 4>(posb, p, a, s);
  else
    dispatch_pos<FMT, 3>(posb, p, a, s);
}

}  // namespace

extern "C" {

int sz_record_cuda(cudaError_t e);  // sz_misc.cu
int sz_check_params(const sz_params* p, int decode_side);

size_t sz_encode_workspace_bytes(uint64_t n, const sz_params* p) {
  if (!p || p->fmt > SZ_E4M3) return 0;
  const uint64_t tiles = (n + encode_tile_for(p->fmt) - 1) / encode_tile_for(p->fmt);
  return static_cast<size_t>((tiles + 1) * sizeof(uint64_t) + 256);
}

int sz_encode(const void* d_words, uint64_t n, const sz_params* p, const sz_encoded* out,
              void* d_ws, size_t ws_bytes, void* stream) {
  if (int rc = sz_check_params(p, 0)) return rc;
  if (n == 0 || !out || !d_words) return SZ_ECONFIG;
  if ((reinterpret_cast<uintptr_t>(d_words) & 31) || (reinterpret_cast<uintptr_t>(out->d_codes) & 15) ||
      (reinterpret_cast<uintptr_t>(out->d_sm) & 15))
    return SZ_EALIGN;
  if (ws_bytes < sz_encode_workspace_bytes(n, p)) return SZ_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int exp_bits = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 5 : 4);
  const int sm_bits = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 3 : 4);
  const bool chunked = !p->sentinel && !p->abs32;
  const int epv = p->fmt == SZ_BF16 ? 16 : 32;
  const uint64_t tile = encode_tile_for(p->fmt);

  EncodeArgs a{};
  a.words = static_cast<const uint8_t*>(d_words);
  a.n = n;
  a.codes = static_cast<uint8_t*>(out->d_codes);
  a.sm = static_cast<uint8_t*>(out->d_sm);
  a.counts = out->d_counts;
  a.positions = out->d_positions;
  a.values = out->d_values;
  a.n_escapes = out->d_n_escapes;
  a.capacity = out->escape_capacity;
  a.num_tiles = (n + tile - 1) / tile;
  a.states = static_cast<uint64_t*>(d_ws);
  a.tile_counter = reinterpret_cast<unsigned long long*>(a.states + a.num_tiles);
  a.n_chunks = chunked ? (n + p->chunk_size - 1) / p->chunk_size : 0;
  a.codes_len = (n * p->code_bits + 7) / 8;
  a.sm_len = (n * sm_bits + 7) / 8;
  a.chunk = p->chunk_size;
  a.chunk_shift = (p->chunk_size & (p->chunk_size - 1)) == 0 ? __builtin_ctz(p->chunk_size) : -1;
  a.counts_mode = 0;
  if (chunked) {
    if (!out->d_counts) return SZ_ECONFIG;
    a.counts_mode = (tile % p->chunk_size == 0 && p->chunk_size % epv == 0) ? 1 : 2;
  }
  if (a.capacity && (!out->d_values || (!p->sentinel && !out->d_positions))) return SZ_ECONFIG;

  cudaError_t e = cudaMemsetAsync(d_ws, 0, (a.num_tiles + 1) * sizeof(uint64_t), s);
  if (e == cudaSuccess && a.counts_mode == 2)
    e = cudaMemsetAsync(out->d_counts, 0, a.n_chunks * sizeof(uint32_t), s);
  if (e != cudaSuccess) return sz_record_cuda(e);

  const int posb = p->sentinel ? 0 : (p->abs32 ? 4 : (p->chunk_size <= 256 ? 1 : 2));
  switch (p->fmt) {
    case SZ_BF16: dispatch_cb<SZ_BF16>(posb, *p, a, s); break;
    case SZ_E5M2: dispatch_cb<SZ_E5M2>(posb, *p, a, s); break;
    default: dispatch_cb<SZ_E4M3>(posb, *p, a, s); break;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return sz_record_cuda(e);
  if (exp_bits != 8 && a.capacity) {
    if (!out->d_values_packed) return SZ_ECONFIG;
    pack_values_kernel<<<296, kThreads, 0, s>>>(a.values, a.n_escapes, a.capacity, exp_bits,
                                                out->d_values_packed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return sz_record_cuda(e);
  }
  return SZ_OK;
}

}  // extern "C"
