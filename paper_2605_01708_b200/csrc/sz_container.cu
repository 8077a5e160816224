// sz_container.cu — SPLZ container framing on the device.
//
// Replaces container.py:201-215 (container_to_bytes) for sections that live
// in HBM: the byte-identical container — 28-byte header, SZCB codebook
// record (container.py:128-137), then counts | codes | sign-mantissa |
// positions | values (FORMATS.md:65-105) — is assembled in one contiguous
// device buffer without a host round trip.  The escape count M is read from
// device memory (the encoder's d_n_escapes), so the header's M field, the
// positions/values lengths and the values offset are all resolved on the
// GPU: framing can be enqueued right behind sz_encode, and the buffer handed
// to a file writer or one NCCL send.
//
// The dense sections (sizes known from N alone) move with cudaMemcpyAsync;
// the M-dependent tail (header + escape sections, ~0.5% of the payload at
// realistic escape rates) with one small grid-stride kernel.
#include "sz_common.cuh"

namespace sz {

constexpr int kPrefixMax = 28 + 9 + 16;  // header + codebook record, <= 16 entries

struct FrameTail {
  uint8_t prefix[kPrefixMax];
  uint32_t prefix_len;
  uint8_t* out;
  uint64_t capacity;
  uint64_t pos_off;          // container offset of the positions section
  const uint8_t* positions;  // M * pos_bytes
  const uint8_t* values;     // ceil(M * exp_bits / 8) (raw bytes for BF16)
  uint32_t pos_bytes;
  uint32_t exp_bits;
  const uint64_t* m_ptr;
  uint64_t m_cap;            // escapes actually stored (encoder capacity)
  uint64_t* nbytes;          // out: total container length
};

__global__ void frame_tail_kernel(const FrameTail t) {
  const uint64_t m = min(*t.m_ptr, t.m_cap);
  const uint64_t pos_len = m * t.pos_bytes;
  const uint64_t val_len = (m * t.exp_bits + 7) / 8;
  const uint64_t total = t.pos_off + pos_len + val_len;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (tid == 0) *t.nbytes = t.pos_off + *t.m_ptr * t.pos_bytes +
                            (*t.m_ptr * t.exp_bits + 7) / 8;
  // header + codebook record, with the escape count patched in (bytes 20-27)
  for (uint64_t i = tid; i < t.prefix_len; i += stride) {
    uint8_t b = t.prefix[i];
    if (i >= 20 && i < 28) b = static_cast<uint8_t>(*t.m_ptr >> (8 * (i - 20)));
    if (i < t.capacity) t.out[i] = b;
  }
  for (uint64_t i = tid; i < pos_len + val_len; i += stride) {
    const uint64_t o = t.pos_off + i;
    if (o >= t.capacity || o >= total) break;
    t.out[o] = i < pos_len ? t.positions[i] : t.values[i - pos_len];
  }
}

}  // namespace sz

extern "C" {

int sz_record_cuda(cudaError_t e);  // sz_misc.cu
int sz_check_params(const sz_params* p, int decode_side);

size_t sz_container_prefix_bytes(const sz_params* p) {
  return p ? 28 + 9 + p->n_entries : 0;
}

uint64_t sz_container_bytes(uint64_t n, uint64_t m, const sz_params* p) {
  if (!p) return 0;
  const uint64_t cb = p->code_bits;
  const uint64_t smb = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 3 : 4);
  const uint64_t eb = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 5 : 4);
  const bool chunked = !p->sentinel && !p->abs32;
  const uint64_t pb = p->sentinel ? 0 : (p->abs32 ? 4 : (p->chunk_size <= 256 ? 1 : 2));
  uint64_t total = sz_container_prefix_bytes(p);
  if (chunked) total += 4 * ((n + p->chunk_size - 1) / p->chunk_size);
  total += (n * cb + 7) / 8;
  total += (n * smb + 7) / 8;
  total += m * pb + (m * eb + 7) / 8;
  return total;
}

int sz_frame_container(const sz_params* p, uint64_t n, const sz_encoded* enc,
                       uint8_t* d_out, uint64_t out_capacity, uint64_t* d_nbytes,
                       void* stream) {
  if (int rc = sz_check_params(p, 0)) return rc;
  if (n == 0 || !enc || !d_out || !d_nbytes || !enc->d_n_escapes || p->n_entries > 16)
    return SZ_ECONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool chunked = !p->sentinel && !p->abs32;
  const uint64_t smb = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 3 : 4);
  const uint32_t eb = p->fmt == SZ_BF16 ? 8 : (p->fmt == SZ_E5M2 ? 5 : 4);
  const uint32_t pb = p->sentinel ? 0 : (p->abs32 ? 4 : (p->chunk_size <= 256 ? 1 : 2));
  const uint8_t* values = eb == 8 ? enc->d_values : enc->d_values_packed;
  if (enc->escape_capacity && !values) return SZ_ECONFIG;

  sz::FrameTail t{};
  // container header (container.py:201-212) + codebook record (:128-137)
  uint8_t* h = t.prefix;
  h[0] = 'S'; h[1] = 'P'; h[2] = 'L'; h[3] = 'Z';
  h[4] = 1;
  h[5] = static_cast<uint8_t>(p->fmt);
  h[6] = p->sentinel ? 1 : (p->abs32 ? 2 : 0);
  h[7] = static_cast<uint8_t>(p->code_bits);
  for (int i = 0; i < 4; ++i) h[8 + i] = static_cast<uint8_t>(p->chunk_size >> (8 * i));
  for (int i = 0; i < 8; ++i) h[12 + i] = static_cast<uint8_t>(n >> (8 * i));
  // bytes 20-27: M, patched on the device
  h[28] = 'S'; h[29] = 'Z'; h[30] = 'C'; h[31] = 'B';
  h[32] = 1;
  h[33] = static_cast<uint8_t>(p->fmt);
  h[34] = static_cast<uint8_t>(p->code_bits);
  h[35] = p->sentinel ? 1 : 0;
  h[36] = static_cast<uint8_t>(p->n_entries);
  for (uint32_t i = 0; i < p->n_entries; ++i) h[37 + i] = p->dec_lut[i];
  t.prefix_len = 37 + p->n_entries;

  const uint64_t counts_len = chunked ? 4 * ((n + p->chunk_size - 1) / p->chunk_size) : 0;
  const uint64_t codes_len = (n * p->code_bits + 7) / 8;
  const uint64_t sm_len = (n * smb + 7) / 8;
  uint64_t off = t.prefix_len;
  const struct { const void* src; uint64_t len; } dense[3] = {
      {enc->d_counts, counts_len}, {enc->d_codes, codes_len}, {enc->d_sm, sm_len}};
  for (const auto& d : dense) {
    if (d.len) {
      if (!d.src) return SZ_ECONFIG;
      if (off + d.len > out_capacity) return SZ_EOUTPUT;
      const cudaError_t e = cudaMemcpyAsync(d_out + off, d.src, d.len,
                                            cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return sz_record_cuda(e);
    }
    off += d.len;
  }
  t.out = d_out;
  t.capacity = out_capacity;
  t.pos_off = off;
  t.positions = static_cast<const uint8_t*>(enc->d_positions);
  t.values = values;
  t.pos_bytes = pb;
  t.exp_bits = eb;
  t.m_ptr = enc->d_n_escapes;
  t.m_cap = enc->escape_capacity;
  t.nbytes = d_nbytes;
  sz::frame_tail_kernel<<<148, sz::kThreads, 0, s>>>(t);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

}  // extern "C"
