"""CPU baseline harness — TEST/BENCH INFRASTRUCTURE ONLY.

Times the oracle (the numpy restatement of the reference codec, sz_oracle.py)
on host cores for ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference``
arm.  Each worker process encodes + decodes its own chunk-aligned shard of the
same synthetic workload (per-shard sections concatenate to the global
encoding in chunk-relative mode, so this is the reference's work split across
processes — a harness, not reference behaviour; the reference itself runs on
one core).  Imports numpy only (spawn-safe, no torch/CUDA in workers).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from oracle import sz_oracle as O


def synth_words(fmt: int, n: int, seed: int, book_w, escapes, rate: float) -> np.ndarray:
    """Sampled-mode words with the bench's exponent distribution."""
    rng = np.random.default_rng(seed)
    exps = np.array([e for e, _ in book_w] + list(escapes), dtype=np.uint8)
    w = np.array([x for _, x in book_w], dtype=np.float64)
    p = np.concatenate([(1 - rate) * w / w.sum(), np.full(len(escapes), rate / len(escapes))])
    e = rng.choice(exps, size=n, p=p / p.sum())
    sm = rng.integers(0, 1 << O.FORMATS[fmt][2], size=n, dtype=np.uint8)
    return O.join(e, sm, fmt)


def _worker(args):
    fmt, n, seed, book, book_w, escapes, rate, chunk, passes = args
    words = synth_words(fmt, n, seed, book_w, escapes, rate)
    p = O.Params(fmt, 4, False, chunk, False)
    t_enc = t_dec = 0.0
    for _ in range(passes):
        t0 = time.perf_counter()
        sec = O.encode(words, p, book)
        t1 = time.perf_counter()
        out = O.decode(sec, p, book)
        t2 = time.perf_counter()
        t_enc += t1 - t0
        t_dec += t2 - t1
    assert np.array_equal(out, words)
    return n * (O.FORMATS[fmt][0] // 8) * passes, t_enc, t_dec


def roundtrip_throughput(fmt: int, book, book_w, escapes, rate: float, chunk: int,
                         n_per_worker: int, workers: int, passes: int = 1,
                         seed: int = 1234) -> dict:
    """Parallel oracle round trip; GB/s of raw input = total bytes / wall time."""
    jobs = [(fmt, n_per_worker, seed + i, tuple(book), tuple(book_w), tuple(escapes), rate,
             chunk, passes) for i in range(workers)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        pool.map(_noop, range(workers))  # warm the pool (imports) outside the clock
        t0 = time.perf_counter()
        res = pool.map(_worker, jobs)
        wall = time.perf_counter() - t0
    total = sum(r[0] for r in res)
    enc = max(r[1] for r in res)
    dec = max(r[2] for r in res)
    # Workers run concurrently: the codec wall time is the slowest worker's
    # encode+decode time (input generation is excluded from the clock).
    codec_wall = max(r[1] + r[2] for r in res)
    return {"gbs": total / codec_wall / 1e9, "bytes": total, "wall_s": codec_wall,
            "wall_with_gen_s": wall,
            "encode_gbs": total / enc / 1e9 if enc else None,
            "decode_gbs": total / dec / 1e9 if dec else None,
            "cpu_seconds": sum(r[1] + r[2] for r in res)}


def _noop(_):
    return os.getpid()


def slice_parity(words: np.ndarray, fmt: int, book, chunk: int, sections: dict) -> bool:
    """Oracle encode of a chunk-aligned prefix == the GPU's global sections
    restricted to those chunks (SURVEY §8c parity method for large configs)."""
    ref = O.encode(words, O.Params(fmt, 4, False, chunk, False), book)
    k = ref["chunk_counts"].size
    m = int(ref["m"])
    return (ref["packed_codes"] == sections["packed_codes"][:len(ref["packed_codes"])]
            and ref["sign_mantissa"] == sections["sign_mantissa"][:len(ref["sign_mantissa"])]
            and np.array_equal(ref["chunk_counts"], sections["chunk_counts"][:k])
            and int(sections["chunk_counts"][:k].sum()) == m
            and np.array_equal(ref["escape_positions"], sections["escape_positions"][:m])
            and np.array_equal(ref["escape_values"], sections["escape_values"][:m]))
