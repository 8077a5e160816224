// sz_encode.cu — K2: single-pass SplitZip encoder for sm_100a.
//
// Replaces codec.py:299-321 (encode) and its byte-identical Quad64 variant
// codec.py:324-401 (encode_quad).
//
// Persistent, warp-specialised kernel (two CTAs per SM, 10 warps each):
//
//   warp 8  PRODUCER  claims tiles (global atomic counter, so tile ids are
//                     handed out in order to running CTAs => look-back
//                     forward progress) and streams each 16 KiB tile of input
//                     words into a shared-memory ring with a 1-D TMA bulk copy
//                     (cp.async.bulk -> UBLKCP), completion on an mbarrier.
//   warps 0-7 DENSE   per 32-byte slot (16 BF16 / 32 FP8 words): split fields
//                     with byte permutes, exponent -> marked code through the
//                     shared-memory LUT (bit 4 = escape, as encode_quad's
//                     marked table codec.py:340-342), pack the 4-bit nibble /
//                     3-bit LE code plane and the sign|mantissa plane (byte
//                     plane for BF16, 3/4-bit LE stream for FP8), vector-store
//                     both, and leave the slot's escape bitmask in smem.
//   warp 9    SCAN    per tile: popc of the slot masks, warp scan, decoupled
//                     look-back over the tile-state array for the global
//                     escape ordinal, per-chunk counts (codec.py:292-295),
//                     then writes every escape's (position, raw exponent)
//                     record in ascending element order and frees the stage.
//
// The look-back latency is hidden behind the ring: the dense warps keep
// streaming later tiles while the scan warp waits on predecessors.
#include "sz_common.cuh"

namespace sz {

constexpr int kEncStages = 4;
constexpr int kEncItems = 2;                           // slots per dense thread
constexpr int kEncSlots = kEncItems * kThreads;        // 512 slots per tile
constexpr int kEncTileBytes = kEncSlots * 32;          // 16 KiB of input words
constexpr int kEncThreads = kThreads + 64;             // + producer + scan warps
constexpr int kProducerWarp = kWarps;                  // warp 8
constexpr int kScanWarp = kWarps + 1;                  // warp 9

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
  int32_t counts_mode;   // 0 none, 1 direct from the scan, 2 atomics (pre-zeroed)
};

struct EncSmem {
  alignas(128) uint8_t in[kEncStages][kEncTileBytes];
  uint32_t fmask[kEncStages][kEncSlots];
  uint32_t pref[kEncSlots + 1];
  uint64_t meta[kEncStages];
  uint64_t full[kEncStages];
  uint64_t computed[kEncStages];
  uint64_t empty[kEncStages];
  uint8_t lut[256];
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

template <int FMT>
__device__ __forceinline__ uint32_t raw_exponent(uint32_t word) {
  if constexpr (FMT == SZ_BF16) return (word >> 7) & 0xFF;
  else if constexpr (FMT == SZ_E5M2) return (word >> 2) & 0x1F;
  else return (word >> 3) & 0x0F;
}

// Dense transform of one 32-byte slot; returns the slot's escape bitmask.
template <int FMT, int CB>
__device__ __forceinline__ uint32_t encode_slot(const uint32_t (&x)[8], const uint8_t* lut,
                                                int nv, const EncodeArgs& a, uint64_t e0) {
  constexpr int EPV = kEpv<FMT>;
  constexpr int G = EPV / 4;
  constexpr int SMB = Fmt<FMT>::kSmBits;
  constexpr int CBYTES = EPV * CB / 8;
  constexpr int SBYTES = EPV * SMB / 8;
  constexpr int CWORDS = (CBYTES + 3) / 4;
  constexpr int SWORDS = (SBYTES + 3) / 4;
  uint32_t mk[G], ag[G];
  uint32_t any = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    uint32_t e4, a4;
    split_group<FMT>(x, g, e4, a4);
    uint32_t m4 = lut4(lut, e4);
    if (nv < EPV) {  // tail slot: zero codes, flags and SM beyond N
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
  if (nv == EPV) {
    st_packed<CBYTES>(a.codes + coff, cw);
    st_packed<SBYTES>(a.sm + soff, sw);
  } else if (nv > 0) {
    st_bytes_clipped<CBYTES>(a.codes, coff, cw, a.codes_len);
    st_bytes_clipped<SBYTES>(a.sm, soff, sw, a.sm_len);
  }
  return fm;
}

template <int FMT, int CB, int POSB>
__global__ void __launch_bounds__(kEncThreads, 2)
    encode_kernel(const __grid_constant__ sz_params p, const EncodeArgs a) {
  constexpr int EPV = kEpv<FMT>;
  constexpr int WB = Fmt<FMT>::kWordBytes;
  constexpr uint64_t TILE = static_cast<uint64_t>(kEncSlots) * EPV;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  EncSmem& S = *reinterpret_cast<EncSmem*>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t n = a.n;
  for (int i = tid; i < 256; i += kEncThreads) S.lut[i] = p.enc_lut[i];
  if (tid == 0) {
    for (int s = 0; s < kEncStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.computed[s], kThreads);
      mbar_init(&S.empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const uint32_t s = it % kEncStages, ph = (it / kEncStages) & 1;
        mbar_wait(&S.empty[s], ph ^ 1);
        const uint64_t tile = atomicAdd(a.tile_counter, 1ull);
        if (tile >= a.num_tiles) {
          S.meta[s] = ~0ull;
          mbar_arrive(&S.full[s]);
          break;
        }
        S.meta[s] = tile;
        const uint64_t e0 = tile * TILE;
        const uint32_t full_slots = static_cast<uint32_t>(min(n - e0, TILE) / EPV);
        const uint32_t bytes = full_slots * 32;
        if (bytes) {
          mbar_arrive_tx(&S.full[s], bytes);
          tma_load_1d(S.in[s], a.words + e0 * WB, bytes, &S.full[s]);
        } else {
          mbar_arrive(&S.full[s]);
        }
      }
    }
    return;
  }

  if (warp < kWarps) {
    // ------------------------------------------------------------ dense warps
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it % kEncStages, ph = (it / kEncStages) & 1;
      mbar_wait(&S.full[s], ph);
      const uint64_t tile = S.meta[s];
      if (tile == ~0ull) break;
      const uint64_t tile_e0 = tile * TILE;
#pragma unroll
      for (int i = 0; i < kEncItems; ++i) {
        const int slot = i * kThreads + tid;
        const uint64_t e0 = tile_e0 + static_cast<uint64_t>(slot) * EPV;
        const int nv = e0 + EPV <= n ? EPV : (e0 < n ? static_cast<int>(n - e0) : 0);
        uint32_t x[8];
        if (nv == EPV) {
          const uint4* src = reinterpret_cast<const uint4*>(S.in[s] + slot * 32);
          const uint4 v0 = src[0], v1 = src[1];
          x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
          x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
        } else {
          ld_bytes_clipped<32>(a.words, e0 * WB, x, nv > 0 ? n * WB : 0);
        }
        S.fmask[s][slot] = encode_slot<FMT, CB>(x, S.lut, nv, a, e0);
      }
      mbar_arrive(&S.computed[s]);
    }
    return;
  }

  // ---------------------------------------------------------------- scan warp
  constexpr int SPL = kEncSlots / 32;  // 16 consecutive slots per lane
  for (uint32_t it = 0;; ++it) {
    const uint32_t s = it % kEncStages, ph = (it / kEncStages) & 1;
    mbar_wait(&S.full[s], ph);
    const uint64_t tile = S.meta[s];
    if (tile == ~0ull) break;
    mbar_wait(&S.computed[s], ph);
    const uint64_t tile_e0 = tile * TILE;

    uint32_t msk[SPL];
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      msk[j] = S.fmask[s][lane * SPL + j];
      cnt += __popc(msk[j]);
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint64_t tile_excl = lookback_warp(a.states, tile, total);
    if (lane == 0 && tile == a.num_tiles - 1) *a.n_escapes = tile_excl + total;

    if (a.counts_mode == 1) {
      // chunks tile the CTA tile: count = difference of slot prefixes
      uint32_t run = incl - cnt;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        run += __popc(msk[j]);
        S.pref[lane * SPL + j + 1] = run;
      }
      if (lane == 0) S.pref[0] = 0;
      __syncwarp();
      const uint32_t spc = a.chunk / EPV;
      const uint32_t chunks_here = static_cast<uint32_t>(TILE / a.chunk);
      const uint64_t k_base = tile_e0 / a.chunk;
      for (uint32_t k = lane; k < chunks_here && k_base + k < a.n_chunks; k += 32)
        a.counts[k_base + k] = S.pref[(k + 1) * spc] - S.pref[k * spc];
    }
    bool per_escape_atomics = false;
    if (a.counts_mode == 2) {
      const uint64_t last = min(tile_e0 + TILE, n) - 1;
      const uint64_t k0 = tile_e0 / a.chunk;
      if (k0 == last / a.chunk) {
        if (lane == 0 && total) atomicAdd(&a.counts[k0], total);
      } else {
        per_escape_atomics = true;
      }
    }

    if (total) {
      uint64_t ord = tile_excl + incl - cnt;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        uint32_t m = msk[j];
        const uint32_t slot = lane * SPL + j;
        const uint64_t e0 = tile_e0 + static_cast<uint64_t>(slot) * EPV;
        const bool in_smem = e0 + EPV <= n;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          const uint64_t idx = e0 + b;
          uint32_t word;
          if (in_smem) {
            const uint8_t* w = S.in[s] + (slot * EPV + b) * WB;
            word = WB == 2 ? *reinterpret_cast<const uint16_t*>(w) : *w;
          } else {
            word = WB == 2 ? reinterpret_cast<const uint16_t*>(a.words)[idx] : a.words[idx];
          }
          if (ord < a.capacity) {
            a.values[ord] = static_cast<uint8_t>(raw_exponent<FMT>(word));
            if constexpr (POSB == 4) {
              static_cast<uint32_t*>(a.positions)[ord] = static_cast<uint32_t>(idx);
            } else if constexpr (POSB == 2 || POSB == 1) {
              const uint64_t pos =
                  a.chunk_shift >= 0 ? (idx & (a.chunk - 1)) : (idx % a.chunk);
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
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[s]);
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

uint64_t encode_tile_for(uint32_t fmt) {
  return static_cast<uint64_t>(kEncSlots) * (fmt == SZ_BF16 ? 16 : 32);
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int FMT, int CB, int POSB>
cudaError_t launch_encode(const sz_params& p, const EncodeArgs& a, cudaStream_t s) {
  auto kern = encode_kernel<FMT, CB, POSB>;
  const int smem = static_cast<int>(sizeof(EncSmem));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kEncThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const uint64_t want = static_cast<uint64_t>(sm_count()) * per_sm;
  const unsigned grid = static_cast<unsigned>(a.num_tiles < want ? a.num_tiles : want);
  kern<<<grid, kEncThreads, smem, s>>>(p, a);
  return cudaGetLastError();
}

template <int FMT, int CB>
cudaError_t dispatch_pos(int posb, const sz_params& p, const EncodeArgs& a, cudaStream_t s) {
  switch (posb) {
    case 0: return launch_encode<FMT, CB, 0>(p, a, s);
    case 1: return launch_encode<FMT, CB, 1>(p, a, s);
    case 2: return launch_encode<FMT, CB, 2>(p, a, s);
    default: return launch_encode<FMT, CB, 4>(p, a, s);
  }
}

template <int FMT>
cudaError_t dispatch_cb(int posb, const sz_params& p, const EncodeArgs& a, cudaStream_t s) {
  return p.code_bits == 4 ? dispatch_pos<FMT, 4>(posb, p, a, s)
                          : dispatch_pos<FMT, 3>(posb, p, a, s);
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
  if ((reinterpret_cast<uintptr_t>(d_words) & 31) ||
      (reinterpret_cast<uintptr_t>(out->d_codes) & 15) ||
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
    case SZ_BF16: e = dispatch_cb<SZ_BF16>(posb, *p, a, s); break;
    case SZ_E5M2: e = dispatch_cb<SZ_E5M2>(posb, *p, a, s); break;
    default: e = dispatch_cb<SZ_E4M3>(posb, *p, a, s); break;
  }
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
