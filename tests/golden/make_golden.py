"""Generate golden vectors by running the REAL reference package.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It copies ``/root/reference/pkg/src`` to a scratch dir, imports ``splitzip``
from there, and records, for a matrix of inputs and codec configs, every
payload section the reference ``encode`` produces, its ``decode`` output,
``build_histogram``/``select_codebook`` results, the reference's size
formulas, and the exception class + ``chunk`` for a set of corrupted
streams.  Output: ``tests/golden/golden.npz`` + ``tests/golden/manifest.json``
(small; committed).  Nothing on the GPU box reads ``/root/reference``.
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def load_reference():
    scratch = Path(tempfile.mkdtemp(prefix="szref_"))
    shutil.copytree("/root/reference/pkg/src/splitzip", scratch / "splitzip")
    sys.path.insert(0, str(scratch))
    import splitzip  # noqa: E402
    return splitzip


def main():
    sz = load_reference()
    from splitzip.codec import EncodedStreams
    from splitzip import container as ref_container

    BF16, E5M2, E4M3 = (sz.ElementFormat.BF16, sz.ElementFormat.FP8_E5M2,
                        sz.ElementFormat.FP8_E4M3)
    FMT_ID = {BF16: 0, E5M2: 1, E4M3: 2}
    EXPL, SENT = sz.CodebookMode.TOPK_EXPLICIT, sz.CodebookMode.TOP15_SENTINEL
    CHUNK, ABS = sz.PositionMode.CHUNK_RELATIVE, sz.PositionMode.ABSOLUTE_32

    arrays: dict[str, np.ndarray] = {}
    cases: list[dict] = []

    def rand(fmt, n, seed):
        rng = np.random.default_rng(seed)
        return rng.integers(0, 1 << fmt.word_bits, size=n).astype(fmt.word_dtype)

    def exact(fmt, n, rate, seed, book, esc):
        return sz.generate(sz.ExponentSpec(fmt, count=n, seed=seed, in_book=book,
                                           escape_values=esc, escape_rate=rate,
                                           exact_counts=True)).words

    def record(cid, fmt, words, code_bits=4, mode=EXPL, chunk=1024, pos=CHUNK,
               book=None, tag=""):
        stream = sz.RawTensorStream(fmt, np.asarray(words, dtype=fmt.word_dtype))
        cb = (sz.ExponentCodebook(fmt, tuple(book), code_bits, mode)
              if book is not None else None)
        cfg = sz.CodecConfig(fmt, code_bits, mode, chunk, pos, cb)
        enc = sz.encode(stream, cfg)
        quad = sz.encode_quad(stream, cfg)
        assert enc.packed_codes == quad.packed_codes
        dec = sz.decode(enc, cfg, enc.codebook)
        assert np.array_equal(dec.words, stream.words)
        secs = dict(enc.section_bytes())
        hist = sz.build_histogram(stream)
        p = f"{cid}/"
        arrays[p + "words"] = stream.words
        arrays[p + "hist"] = hist.counts
        for name, data in secs.items():
            arrays[p + name] = np.frombuffer(data, dtype=np.uint8)
        arrays[p + "escape_values_raw"] = np.asarray(enc.escape_values, np.uint8)
        # the reference's SPLZ container bytes (container.py:201-215)
        arrays[p + "container"] = np.frombuffer(
            ref_container.container_to_bytes(enc, cfg, enc.codebook), dtype=np.uint8)
        cases.append({
            "id": cid, "tag": tag, "fmt": FMT_ID[fmt], "code_bits": code_bits,
            "sentinel": mode is SENT, "chunk": chunk, "abs32": pos == ABS,
            "pinned": book is not None, "book": list(enc.codebook.entries),
            "n": enc.n_elements, "m": enc.n_escapes,
            "payload_nbytes": enc.payload_nbytes,
            "formula_payload": sz.compressed_payload_bytes(enc.n_elements, enc.n_escapes, cfg),
            "formula_ratio": sz.compression_ratio(enc.n_elements, enc.n_escapes, cfg),
            "pos_dtype": str(enc.escape_positions.dtype),
            "entropy": sz.entropy_bits(hist),
            "top8": sz.top_k_coverage(hist, 8),
            "top16": sz.top_k_coverage(hist, min(16, fmt.exp_bins)),
        })
        return enc, cfg

    # 1. SURVEY §8(a') known answers.
    record("ka_bf16", BF16, [0x3F80, 0xBF80, 0x0800, 0x4000, 0x3F81], book=(0x7F, 0x80),
           tag="known-answer")
    record("ka_e5m2", E5M2, [0x23, 0xA5, 0x82], book=(8, 9), tag="known-answer")

    # 2. The reference's 36-config universal matrix (test_codec.py:40-51) on
    #    uniform random words, dynamic codebook.
    idx = 0
    for fmt in (BF16, E5M2, E4M3):
        for cb in (3, 4):
            for mode, pos in ((EXPL, CHUNK), (EXPL, ABS), (SENT, CHUNK)):
                for chunk in (256, 1024):
                    record(f"mat{idx:02d}", fmt, rand(fmt, 3001, idx), cb, mode, chunk, pos,
                           tag="matrix")
                    idx += 1

    # 3. Realistic exact-count profiles with pinned codebooks.
    B16 = tuple((0x70 + i, 0.72 ** i) for i in range(16))
    B15 = B16[:15]
    B8 = tuple((0x74 + i, 0.72 ** i) for i in range(8))
    EB = tuple(range(0x10, 0x18))
    E16 = tuple((8 + i, 0.72 ** i) for i in range(16))
    E8 = E16[:8]
    EE = (0, 1, 2, 3, 28, 29, 30, 31)
    F8 = tuple((4 + i, 0.72 ** i) for i in range(8))
    FE = (0, 1, 2, 3, 12, 13, 14, 15)
    ent = lambda b: [e for e, _ in b]
    for rate in (0.0, 0.0016, 0.0123, 0.0789):
        r = int(rate * 1e4)
        record(f"kv_bf16_r{r}", BF16, exact(BF16, 20_000, rate, 3, B16, EB), book=ent(B16),
               tag="profile")
        record(f"kv_e5m2_r{r}", E5M2, exact(E5M2, 20_000, rate, 4, E16, EE), book=ent(E16),
               tag="profile")
    record("kv_bf16_top8", BF16, exact(BF16, 30_000, 0.0789, 5, B8, EB), 3, book=ent(B8),
           tag="profile")
    record("kv_bf16_sent", BF16, exact(BF16, 30_000, 0.0027, 6, B15, EB), 4, SENT,
           book=ent(B15), tag="profile")
    record("kv_e5m2_top8", E5M2, exact(E5M2, 30_000, 0.0772, 7, E8, EE), 3, book=ent(E8),
           tag="profile")
    record("kv_e4m3_top8", E4M3, exact(E4M3, 30_000, 0.0783, 8, F8, FE), 3, book=ent(F8),
           tag="profile")
    record("kv_bf16_abs32", BF16, exact(BF16, 30_000, 0.01, 9, B16, EB), 4, EXPL, 1024, ABS,
           book=ent(B16), tag="profile")

    # 4. Boundary lengths (quad tail, odd nibble, partial chunks).
    for n in (1, 2, 3, 4, 5, 7, 15, 16, 17, 31, 33, 1023, 1024, 1025, 4097, 8191, 8193):
        record(f"len_bf16_{n}", BF16, rand(BF16, n, 1000 + n), tag="length")
        record(f"len_e5m2_{n}", E5M2, rand(E5M2, n, 2000 + n), tag="length")

    # 5. Chunk-size sweep, including non powers of two and chunks > tile.
    for c in (1, 3, 32, 100, 1000, 2048, 4096, 16384, 65536):
        n = 140_001 if c >= 16384 else 20_001
        record(f"chunk_bf16_{c}", BF16, exact(BF16, n, 0.05, 11, B16, EB), chunk=c,
               book=ent(B16), tag="chunk")
        record(f"chunk_e5m2_{c}", E5M2, exact(E5M2, n, 0.05, 12, E16, EE), chunk=c,
               book=ent(E16), tag="chunk")

    # 6. Zero-coverage codebook: every element escapes (test_codec.py:241-249).
    record("allesc_bf16", BF16, exact(BF16, 4096, 0.0, 14, B16, EB), book=(0x01, 0x02),
           tag="all-escape")
    record("allesc_e5m2", E5M2, exact(E5M2, 4099, 0.0, 15, E16, EE), book=(0x1F,),
           tag="all-escape")
    # NaN/Inf are opaque bit patterns (test_codec.py:251-254).
    record("naninf", BF16, [0x7FC0, 0x7F80, 0xFF80, 0xFFFF, 0x0001], tag="nan-inf")

    # 7. Corruption verdicts: mutate one section of a valid encode and record
    #    the reference's exception class and chunk.
    corrupt = []
    base_words = exact(BF16, 3000, 0.01, 12, B16, EB)
    stream = sz.RawTensorStream(BF16, base_words)
    cfg = sz.CodecConfig(BF16, codebook=sz.select_codebook(
        sz.build_histogram(stream), 4, EXPL))
    enc = sz.encode(stream, cfg)
    arrays["corrupt/words"] = base_words
    first_escape = int(np.repeat(np.arange(enc.chunk_counts.size) * 1024,
                                 enc.chunk_counts)[0] + enc.escape_positions[0])

    def mutate(cid, **fields):
        kw = dict(n_elements=enc.n_elements, n_escapes=enc.n_escapes,
                  packed_codes=enc.packed_codes, sign_mantissa=enc.sign_mantissa,
                  chunk_counts=enc.chunk_counts, escape_positions=enc.escape_positions,
                  escape_values=enc.escape_values, codebook=enc.codebook)
        kw.update(fields)
        bad = EncodedStreams(**kw)
        try:
            sz.decode(bad, cfg, enc.codebook)
            verdict = {"raised": None, "chunk": None}
        except sz.SplitZipError as exc:
            verdict = {"raised": type(exc).__name__, "chunk": getattr(exc, "chunk", None)}
        p = f"corrupt_{cid}/"
        arrays[p + "packed_codes"] = np.frombuffer(kw["packed_codes"], np.uint8)
        arrays[p + "sign_mantissa"] = np.frombuffer(kw["sign_mantissa"], np.uint8)
        arrays[p + "chunk_counts"] = np.asarray(kw["chunk_counts"], np.uint32)
        arrays[p + "escape_positions"] = np.asarray(kw["escape_positions"])
        arrays[p + "escape_values"] = np.asarray(kw["escape_values"], np.uint8)
        corrupt.append({"id": cid, "n": kw["n_elements"], "m": kw["n_escapes"], **verdict})

    pos = enc.escape_positions.copy()
    pos[3] = 1024
    mutate("pos_over_chunk", escape_positions=pos)
    vals = enc.escape_values.copy()
    vals[5] = enc.codebook.entries[0]
    mutate("value_in_book", escape_values=vals)
    mutate("n_plus_one", n_elements=enc.n_elements + 1)
    pos = enc.escape_positions.copy()
    c0 = int(enc.chunk_counts[0])
    pos[c0:c0 + 2] = pos[c0:c0 + 2][::-1]
    mutate("not_increasing", escape_positions=pos)
    codes = bytearray(enc.packed_codes)
    bi, lo = divmod(first_escape, 2)
    codes[bi] |= 0x05 if lo == 0 else 0x50
    mutate("nondummy", packed_codes=bytes(codes))
    cnt = enc.chunk_counts.copy()
    cnt[1] += 1
    mutate("counts_total", chunk_counts=cnt)
    cnt = enc.chunk_counts.copy()
    cnt[0] += 1
    cnt[1] -= 1
    mutate("counts_shift", chunk_counts=cnt)
    pos = enc.escape_positions.copy()
    pos[-1] = 1023
    mutate("past_end", escape_positions=pos)
    codes = bytearray(enc.packed_codes)
    mutate("short_codes", packed_codes=bytes(codes[:-1]))
    mutate("m_too_big", n_escapes=enc.n_elements + 1)
    vals = enc.escape_values.copy()
    mutate("m_mismatch", escape_values=vals[:-1])
    mutate("clean")

    # 7b. Corruption verdicts of the other modes: abs32 positions, sentinel
    #     marks, E5M2 values (5-bit domain), 3-bit codes past a short book.
    bases = {}

    def make_base(bid, fmt, words, code_bits, mode, chunk, pos, book):
        stream = sz.RawTensorStream(fmt, np.asarray(words, dtype=fmt.word_dtype))
        cb = sz.ExponentCodebook(fmt, tuple(book), code_bits, mode)
        bcfg = sz.CodecConfig(fmt, code_bits, mode, chunk, pos, cb)
        benc = sz.encode(stream, bcfg)
        arrays[f"corrupt_base_{bid}/words"] = stream.words
        bases[bid] = {"fmt": FMT_ID[fmt], "code_bits": code_bits, "sentinel": mode is SENT,
                      "chunk": chunk, "abs32": pos is ABS, "book": [int(e) for e in book]}

        def bmutate(cid, **fields):
            kw = dict(n_elements=benc.n_elements, n_escapes=benc.n_escapes,
                      packed_codes=benc.packed_codes, sign_mantissa=benc.sign_mantissa,
                      chunk_counts=benc.chunk_counts, escape_positions=benc.escape_positions,
                      escape_values=benc.escape_values, codebook=benc.codebook)
            kw.update(fields)
            try:
                sz.decode(EncodedStreams(**kw), bcfg, benc.codebook)
                verdict = {"raised": None, "chunk": None}
            except sz.SplitZipError as exc:
                verdict = {"raised": type(exc).__name__, "chunk": getattr(exc, "chunk", None)}
            q = f"corrupt_{cid}/"
            arrays[q + "packed_codes"] = np.frombuffer(kw["packed_codes"], np.uint8)
            arrays[q + "sign_mantissa"] = np.frombuffer(kw["sign_mantissa"], np.uint8)
            arrays[q + "chunk_counts"] = np.asarray(kw["chunk_counts"], np.uint32)
            arrays[q + "escape_positions"] = np.asarray(kw["escape_positions"])
            arrays[q + "escape_values"] = np.asarray(kw["escape_values"], np.uint8)
            corrupt.append({"id": cid, "base": bid, "n": kw["n_elements"],
                            "m": kw["n_escapes"], **verdict})
        return benc, bmutate

    def set_code(packed, i, code, bits):
        buf = bytearray(packed)
        for b in range(bits):
            bit = i * bits + b
            if (code >> b) & 1:
                buf[bit >> 3] |= 1 << (bit & 7)
            else:
                buf[bit >> 3] &= ~(1 << (bit & 7)) & 0xFF
        return bytes(buf)

    b16 = tuple(e for e, _ in B16)
    # abs32 positions (codec.py:500-507)
    benc, bm = make_base("abs", BF16, exact(BF16, 3000, 0.01, 21, B16, EB), 4, EXPL, 1024,
                         ABS, b16)
    pos = benc.escape_positions.copy()
    pos[3], pos[4] = pos[4], pos[3]
    bm("abs_not_increasing", escape_positions=pos)
    pos = benc.escape_positions.copy()
    pos[-1] = benc.n_elements
    bm("abs_past_end", escape_positions=pos)
    vals = benc.escape_values.copy()
    vals[2] = b16[0]
    bm("abs_value_in_book", escape_values=vals)
    bm("abs_m_mismatch", escape_values=benc.escape_values[:-1])
    bm("abs_clean")
    # sentinel marks (codec.py:459-467)
    benc, bm = make_base("sent", BF16, exact(BF16, 3000, 0.01, 22, B16, EB), 4, SENT, 1024,
                         CHUNK, b16[:15])
    codes_u = np.frombuffer(benc.packed_codes, np.uint8)
    nib = np.stack([codes_u & 15, codes_u >> 4], axis=1).reshape(-1)[:benc.n_elements]
    plain = int(np.flatnonzero(nib != 15)[7])
    mark = int(np.flatnonzero(nib == 15)[3])
    bm("sent_extra_mark", packed_codes=set_code(benc.packed_codes, plain, 15, 4))
    bm("sent_lost_mark", packed_codes=set_code(benc.packed_codes, mark, 0, 4))
    vals = benc.escape_values.copy()
    vals[1] = b16[0]
    bm("sent_value_in_book", escape_values=vals)
    bm("sent_clean")
    # E5M2 escape values: 5-bit domain (codec.py:451-457)
    benc, bm = make_base("e5", E5M2, exact(E5M2, 4000, 0.01, 23, E16, EE), 4, EXPL, 1024,
                         CHUNK, tuple(e for e, _ in E16))
    vals = benc.escape_values.copy()
    vals[4] = 40
    bm("e5_value_domain", escape_values=vals)
    vals = benc.escape_values.copy()
    vals[6] = 8
    bm("e5_value_in_book", escape_values=vals)
    pos = benc.escape_positions.copy()
    pos[0] = 1500
    bm("e5_pos_over_chunk", escape_positions=pos)
    bm("e5_clean")
    # 3-bit codes with a 6-entry book: codes 6 and 7 decode nothing
    benc, bm = make_base("tri", BF16, exact(BF16, 3000, 0.01, 24, B16, EB), 3, EXPL, 1024,
                         CHUNK, b16[:6])
    bm("tri_code_range", packed_codes=set_code(benc.packed_codes, 1234, 7, 3))
    bm("tri_clean")

    # 8. Container parse verdicts (container.py:225-296) on mutated bytes of a
    #    valid BF16 container and an E5M2 one (5-bit values section).
    cverdicts = []
    for base_id in ("kv_bf16_r16", "kv_e5m2_r123"):
        good = arrays[f"{base_id}/container"].tobytes()
        k = len(next(c for c in cases if c["id"] == base_id)["book"])
        muts = {
            "clean": good,
            "bad_magic": b"SPLX" + good[4:],
            "bad_version": good[:4] + bytes([2]) + good[5:],
            "bad_format": good[:5] + bytes([7]) + good[6:],
            "bad_mode": good[:6] + bytes([9]) + good[7:],
            "bad_code_bits": good[:7] + bytes([5]) + good[8:],
            "zero_chunk": good[:8] + bytes(4) + good[12:],
            "zero_n": good[:12] + bytes(8) + good[20:],
            "m_gt_n": good[:20] + (10 ** 9).to_bytes(8, "little") + good[28:],
            "bad_cb_magic": good[:28] + b"SZCX" + good[32:],
            "cb_mismatch_bits": good[:34] + bytes([3]) + good[35:],
            "truncated_header": good[:20],
            "truncated_codebook": good[:28 + 9 + k - 1],
            "truncated_counts": good[:28 + 9 + k + 3],
            "truncated_values": good[:-1],
            "trailing": good + b"\x00",
        }
        for mid, data in muts.items():
            try:
                ref_container.container_from_bytes(data)
                verdict = {"raised": None, "section": None}
            except sz.SplitZipError as exc:
                verdict = {"raised": type(exc).__name__,
                           "section": getattr(exc, "section", None)}
            arrays[f"cont_{base_id}_{mid}"] = np.frombuffer(data, dtype=np.uint8)
            cverdicts.append({"id": f"cont_{base_id}_{mid}", "base": base_id, **verdict})

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "manifest.json").write_text(json.dumps(
        {"generator": "tests/golden/make_golden.py (reference splitzip 0.1.0)",
         "cases": cases, "corruptions": corrupt, "corruption_bases": bases,
         "container_verdicts": cverdicts}, indent=1))
    print(f"{len(cases)} cases, {len(corrupt)} corruption verdicts, "
          f"{(HERE / 'golden.npz').stat().st_size} bytes")


if __name__ == "__main__":
    main()
