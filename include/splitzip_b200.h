/*
 * splitzip_b200.h — C ABI of the B200-native SplitZip codec.
 *
 * Plain pointers, sizes and a `void*` CUDA stream; no torch or numpy types.
 * Every pointer named `d_*` is DEVICE memory owned by the caller (the library
 * never allocates or frees caller memory).  Every entry point only enqueues
 * work on `stream` and returns; results that the host needs (escape count,
 * decode status) are written to device memory and read by the caller after
 * its own stream synchronisation.  No hidden global state: concurrent calls
 * on different streams are safe as long as each call has its own workspace.
 *
 * Each entry point cites the reference function it replaces
 * (/root/reference/pkg/src/splitzip/<file>:<line>).  The reference is a
 * pure-Python package whose public functions ARE its plugin interface; the
 * Python mirror in paper_2605_01708_b200/ binds these symbols with ctypes
 * behind the reference's own names and signatures.
 */
#ifndef SPLITZIP_B200_H
#define SPLITZIP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SZ_ABI_VERSION 1

/* Element formats: same numbering as the container's format byte
 * (container.py:278-279). */
enum sz_format { SZ_BF16 = 0, SZ_E5M2 = 1, SZ_E4M3 = 2 };

/* Return codes. */
enum sz_status {
  SZ_OK = 0,
  SZ_ECONFIG = 1,   /* unsupported/inconsistent parameters (ConfigError)     */
  SZ_EWORKSPACE = 2,/* workspace too small                                   */
  SZ_EALIGN = 3,    /* a pointer is not aligned as documented                */
  SZ_ECUDA = 4,     /* a CUDA launch failed (sz_last_cuda_error() has detail) */
  SZ_EOUTPUT = 5    /* an output buffer is too small (sz_frame_container)     */
};

/* Codec parameters = CodecConfig (codec.py:86-135) + the codebook's LUTs
 * (calibration.py:149-158) in kernel-ready form.
 *
 * enc_lut[e] is the "marked" table of encode_quad (codec.py:340-342):
 *   member exponent  -> its code (0..2^code_bits-1)
 *   escape exponent  -> 0x10 | fill, fill = 0 (explicit, DUMMY_CODE codec.py:67)
 *                       or the sentinel code 2^code_bits-1 (sentinel mode).
 * dec_lut[c] = codebook.entries[c] for c < n_entries, 0 above (codec.py:416-418).
 */
typedef struct sz_params {
  uint32_t fmt;        /* enum sz_format                                       */
  uint32_t code_bits;  /* 3 or 4                                               */
  uint32_t sentinel;   /* 0 = TOPK_EXPLICIT, 1 = TOP15_SENTINEL                */
  uint32_t abs32;      /* 1 = PositionMode.ABSOLUTE_32 (explicit mode only)    */
  uint32_t chunk_size; /* >= 1; <= 65536 when chunk-relative                   */
  uint32_t n_entries;  /* codebook length                                      */
  uint8_t enc_lut[256];
  uint8_t dec_lut[16];
} sz_params;

/* Output sections of one encode (EncodedStreams, codec.py:151-188).  Sizes
 * the caller must provide (N elements, C = ceil(N/chunk) chunks when chunked,
 * K = escape capacity):
 *   d_codes      ceil(N*code_bits/8) bytes
 *   d_sm         N (bf16) | ceil(3N/8) (e5m2) | ceil(N/2) (e4m3) bytes
 *   d_counts     C x uint32 (chunked explicit mode only, else may be NULL)
 *   d_positions  K x {u8|u16|u32} (explicit mode only)
 *   d_values     K x uint8 raw exponents, escape order
 *   d_values_packed  ceil(K*exp_bits/8) bytes, FP8 only (may be NULL for BF16)
 *   d_n_escapes  1 x uint64: the true escape count M, written even when
 *                M > K (then only the first K escapes are stored and the
 *                caller re-runs with a larger capacity — SZ overflow protocol).
 * Alignment: d_words 32 B; d_codes, d_sm 16 B.
 */
typedef struct sz_encoded {
  void* d_codes;
  void* d_sm;
  uint32_t* d_counts;
  void* d_positions;
  uint8_t* d_values;
  uint8_t* d_values_packed;
  uint64_t* d_n_escapes;
  uint64_t escape_capacity;
  /* Optional append mode for chunk-aligned pieces of one stream: when
   * non-NULL, this call's escapes are written at ordinals *d_escape_base + i
   * (capacity applies to the absolute ordinal) and *d_escape_base is advanced
   * by this call's M, all on the device — so a piecewise host<->device
   * pipeline builds the global escape stream without host round trips
   * (chunk-relative sections of chunk-aligned pieces concatenate exactly). */
  uint64_t* d_escape_base;
} sz_encoded;

/* Decode inputs: the same sections, read-only, plus the declared counts. */
typedef struct sz_encoded_in {
  const void* d_codes;
  const void* d_sm;
  const uint32_t* d_counts;
  const void* d_positions;
  const uint8_t* d_values;   /* M raw (unpacked) exponent values            */
  uint64_t n_elements;
  uint64_t n_escapes;
  uint64_t n_counts;         /* length of d_counts as supplied              */
  /* Optional: when non-NULL the escape count M is read from this device
   * word (e.g. the encoder's d_n_escapes, or a received header) so a
   * encode->transfer->decode pipeline needs no host round trip.  n_escapes
   * is then the CAPACITY of d_positions / d_values (0 = they hold N entries):
   * a device M above it is clamped for every read and reported as
   * SZ_DEC_CAPACITY in the status flags, so an encoder overflow (M > K, see
   * sz_encoded) never reads past the caller's escape buffers. */
  const uint64_t* d_n_escapes;
} sz_encoded_in;

/* Decode verdict, written to device memory (zero it before the call —
 * sz_decode does this itself on `stream`).  `flags` has one bit per failed
 * check (SZ_DEC_*); first_inv[k] = ~(smallest offending escape ordinal or
 * element index) for check k, 0 if none.  The host maps these to
 * CorruptionError(msg, chunk) in the reference's check order
 * (codec.py:431-476, 491-536). */
enum sz_decode_check {
  SZ_DEC_CODE_PAD = 0,      /* nonzero pad bits in code stream  (codec.py:441-442) */
  SZ_DEC_SM_PAD = 1,        /* nonzero pad bits in 3/4-bit SM   (codec.py:236-237) */
  SZ_DEC_VALUE_DOMAIN = 2,  /* escape value >= exp_bins          (codec.py:451-452) */
  SZ_DEC_VALUE_IN_BOOK = 3, /* escape value is a member          (codec.py:453-457) */
  SZ_DEC_SENTINEL_COUNT = 4,/* sentinel marks != M               (codec.py:461-465) */
  SZ_DEC_ABS_PAST_END = 5,  /* abs32 index >= N                  (codec.py:503-504) */
  SZ_DEC_ABS_NOT_INC = 6,   /* abs32 not strictly increasing     (codec.py:505-506) */
  SZ_DEC_COUNTS_TOTAL = 7,  /* sum(counts) != M                  (codec.py:513-514) */
  SZ_DEC_POS_OVER_CHUNK = 8,/* position >= chunk_size            (codec.py:515-519) */
  SZ_DEC_POS_PAST_END = 9,  /* chunk index >= N                  (codec.py:525-529) */
  SZ_DEC_POS_NOT_INC = 10,  /* not strictly increasing           (codec.py:530-535) */
  SZ_DEC_CODE_RANGE = 11,   /* dense code >= n_entries           (codec.py:408-415) */
  SZ_DEC_NONDUMMY = 12,     /* escape carries a non-dummy code   (codec.py:472-476) */
  SZ_DEC_NUM_CHECKS = 13,
  /* flag only (no first_inv slot): the device-resident M exceeds the escape
   * capacity given in sz_encoded_in.n_escapes */
  SZ_DEC_CAPACITY = 13
};

typedef struct sz_decode_status {
  uint32_t flags;
  uint32_t _pad;
  uint64_t first_inv[SZ_DEC_NUM_CHECKS];
  uint64_t counts_total;   /* sum of chunk counts (chunked mode)            */
  uint64_t marks_total;    /* number of sentinel codes (sentinel mode)      */
} sz_decode_status;

/* ---- library info ------------------------------------------------------ */
int sz_abi_version(void);
const char* sz_last_cuda_error(void);

/* ---- L0 bit primitives (formats.py) ------------------------------------ */
/* split_fields (formats.py:113-133): words -> exponent / sign|mantissa bytes. */
int sz_split_fields(const void* d_words, uint64_t n, uint32_t fmt,
                    uint8_t* d_exp, uint8_t* d_sm, void* stream);
/* reconstruct (formats.py:136-155). */
int sz_reconstruct(const uint8_t* d_exp, const uint8_t* d_sm, uint64_t n,
                   uint32_t fmt, void* d_words, void* stream);
/* pack_codes (formats.py:167-189) for widths 3, 4, 5, 8; symbols must fit
 * (the caller checks range, formats.py:158-163 — sz_max_u8 helps). */
int sz_pack_bits(const uint8_t* d_symbols, uint64_t n, uint32_t width,
                 uint8_t* d_out, void* stream);
/* unpack_codes (formats.py:197-220); *d_pad_nonzero (u32) receives 1 when a
 * pad bit is set (trailing_bits_zero, formats.py:223-231). */
int sz_unpack_bits(const uint8_t* d_packed, uint64_t n, uint32_t width,
                   uint8_t* d_symbols, uint32_t* d_pad_nonzero, void* stream);
/* max over n bytes into *d_max (u32); used for CodeRangeError checks. */
int sz_max_u8(const uint8_t* d_in, uint64_t n, uint32_t* d_max, void* stream);

/* ---- K1 calibration histogram (calibration.py:79-85) ------------------- */
/* d_counts: 2^exp_bits x uint64, overwritten (not accumulated). */
size_t sz_histogram_workspace_bytes(uint64_t n, uint32_t fmt);
int sz_histogram(const void* d_words, uint64_t n, uint32_t fmt, uint64_t* d_counts,
                 void* d_ws, size_t ws_bytes, void* stream);

/* ---- K2 encode (codec.py:299-321 == encode_quad codec.py:324-401) ------ */
size_t sz_encode_workspace_bytes(uint64_t n, const sz_params* p);
int sz_encode(const void* d_words, uint64_t n, const sz_params* p,
              const sz_encoded* out, void* d_ws, size_t ws_bytes, void* stream);

/* ---- K4 decode (codec.py:421-536) --------------------------------------- */
/* m: the escape count the decode will declare (n = size for any M).  For
 * chunk-relative streams with chunk >= 32 and M >= N/50 the workspace also
 * holds the escape-dense path's element bitmap (N/8 bytes) and per-tile
 * counts; sz_decode takes that path only when the workspace it is given is
 * large enough (else the general path, correct for any M). */
size_t sz_decode_workspace_bytes(uint64_t n, uint64_t m, const sz_params* p);
int sz_decode(const sz_encoded_in* in, const sz_params* p, void* d_words_out,
              sz_decode_status* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* Escape-value checks alone (codec.py:446-457) into d_status (zeroed here):
 * used by the host when a later-priority length check already failed. */
int sz_check_values(const uint8_t* d_values, uint64_t m, const sz_params* p,
                    sz_decode_status* d_status, void* stream);

/* ---- K7 bitwise comparison (compare_streams, codec.py:572-581) ---------- */
/* d_result[0] = mismatch count, d_result[1] = ~first mismatch index (0: none). */
int sz_compare(const void* d_a, const void* d_b, uint64_t n, uint32_t word_bytes,
               uint64_t* d_result, void* stream);

/* ---- Paged / segmented streams (paged-KV gather) -------
 * The logical stream is the concatenation of n_segs segments of seg_bytes
 * each (a power of two >= 32; e.g. one vLLM KV-cache block), segment i at
 * the 32-byte-aligned device address d_seg_addrs[i] (a device array of u64).
 * sz_encode_segments reads the blocks in place (the producer warp's bulk
 * copies gather them — no contiguous staging copy), N = n_segs*seg_bytes /
 * word_bytes; its sections are byte-identical to sz_encode of the gathered
 * words.  sz_decode_segments writes the decoded words straight into the
 * destination blocks.  Workspaces as for sz_encode / sz_decode with that N. */
int sz_encode_segments(const uint64_t* d_seg_addrs, uint64_t n_segs, uint64_t seg_bytes,
                       const sz_params* p, const sz_encoded* out, void* d_ws,
                       size_t ws_bytes, void* stream);
/* As sz_encode_segments, given a virtual-address window [va_lo, va_hi) that
 * contains every segment (e.g. the span of the KV-cache tensors) and with
 * every segment 128-byte aligned: full tiles then arrive through a 2-D
 * tensor map over the window (128B-swizzled boxes of min(seg_bytes, 32 KiB)),
 * as the contiguous encoder's do.  Needs seg_bytes >= 1 KiB and a window of
 * < 256 GiB; otherwise (or with va_hi <= va_lo) it is sz_encode_segments.
 * No segment is read outside itself; the window only names addresses. */
int sz_encode_segments_va(const uint64_t* d_seg_addrs, uint64_t n_segs, uint64_t seg_bytes,
                          uint64_t va_lo, uint64_t va_hi, const sz_params* p,
                          const sz_encoded* out, void* d_ws, size_t ws_bytes, void* stream);
int sz_decode_segments(const sz_encoded_in* in, const sz_params* p,
                       const uint64_t* d_seg_addrs, uint64_t n_segs, uint64_t seg_bytes,
                       sz_decode_status* d_status, void* d_ws, size_t ws_bytes,
                       void* stream);

/* ---- Fused encode -> NVLink handoff flags -------------
 * The sender encodes with its sz_encoded outputs pointing INTO the receiver's
 * memory (peer-access / IPC-mapped pointers), so the encoder's own stores
 * carry the compressed sections over NVLink, then sz_peer_signal raises a
 * flag in the receiver's memory (system-scope fence + release store, after
 * every prior kernel on `stream`).  The receiver enqueues sz_peer_wait
 * (system-scope acquire polling until *d_flag >= value) before its decode.
 * A wait gives up after timeout_ns (0 = 30 s) and sets *d_timed_out. */
int sz_peer_signal(uint64_t* d_flag, uint64_t value, void* stream);
int sz_peer_wait(const uint64_t* d_flag, uint64_t value, uint64_t timeout_ns,
                 uint32_t* d_timed_out, void* stream);
/* A dedicated zero-filled device region (cudaMalloc) and its CUDA IPC
 * handle (64 bytes) so another process can map it (sz_ipc_import opens it
 * with lazy peer access: NVLink/NVSwitch between GPUs, plain device memory on
 * the same GPU). */
int sz_device_alloc(uint64_t bytes, void** d_out);
int sz_device_free(void* d);
int sz_ipc_export(const void* d_base, uint8_t* handle_out);
int sz_ipc_import(const uint8_t* handle, void** d_base_out);
int sz_ipc_close(void* d_base);

/* ---- SPLZ container framing (container.py:201-215, FORMATS.md:65-105) ----
 * Byte-identical container = 28-byte header | SZCB codebook record
 * (container.py:128-137) | counts | codes | sign-mantissa | positions |
 * values, assembled in ONE contiguous device buffer from the sections of an
 * encode.  M is read from enc->d_n_escapes on the device (header field,
 * escape section lengths), so framing can be enqueued right behind sz_encode
 * with no host round trip.  *d_nbytes (device u64) receives the container
 * length; the caller sizes d_out with sz_container_bytes(n, capacity, p) and
 * must have encoded with enough escape capacity (M <= enc->escape_capacity).
 * Values come from enc->d_values (BF16) or enc->d_values_packed (FP8). */
size_t sz_container_prefix_bytes(const sz_params* p);          /* 28 + 9 + k */
uint64_t sz_container_bytes(uint64_t n, uint64_t m, const sz_params* p);
int sz_frame_container(const sz_params* p, uint64_t n, const sz_encoded* enc,
                       uint8_t* d_out, uint64_t out_capacity, uint64_t* d_nbytes,
                       void* stream);

/* ---- coverage_by_group (calibration.py:191-212): member count per group -- */
int sz_group_members(const void* d_words, uint64_t n, const sz_params* p,
                     uint64_t group, uint64_t* d_hits, void* stream);

/* ---- K8 synthetic KV generator (bench/test input; distribution of
 * datagen.generate, datagen.py:98-126, sampled mode).  weights_q32[i] is the
 * cumulative probability of exps[i] scaled to 2^32 (last entry 2^32-1). ---- */
int sz_synth_words(void* d_words, uint64_t n, uint32_t fmt, uint64_t seed,
                   const uint8_t* exps, const uint32_t* cdf_q32, uint32_t n_exps,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLITZIP_B200_H */
