"""CPU baseline harness — TEST/BENCH INFRASTRUCTURE ONLY.

Times the oracle (the numpy restatement of the reference codec, sz_oracle.py)
on host cores for ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference``
arm.  Each worker process holds its own chunk-aligned shard of the same
synthetic workload, generated once when the pool starts, and every step
encodes + decodes it (per-shard sections concatenate to the global encoding
in chunk-relative mode, so this is the reference's work split across
processes — a harness, not reference behaviour; the reference itself runs
on one core, which ``one_core`` times on its own).  Imports numpy only
(spawn-safe, no torch/CUDA in workers).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from oracle import sz_oracle as O

_SHARD: dict = {}


def synth_words(fmt: int, n: int, seed: int, book_w, escapes, rate: float) -> np.ndarray:
    """Sampled-mode words with the bench's exponent distribution."""
    rng = np.random.default_rng(seed)
    exps = np.array([e for e, _ in book_w] + list(escapes), dtype=np.uint8)
    w = np.array([x for _, x in book_w], dtype=np.float64)
    p = np.concatenate([(1 - rate) * w / w.sum(), np.full(len(escapes), rate / len(escapes))])
    e = exps[np.searchsorted(np.cumsum(p / p.sum()), rng.random(n), side="right")
             .clip(0, exps.size - 1)]
    sm = rng.integers(0, 1 << O.FORMATS[fmt][2], size=n, dtype=np.uint8)
    return O.join(e, sm, fmt)


def _init(counter, fmt, n, seed, book, book_w, escapes, rate, chunk):
    """Pool initializer: this worker's shard (worker i draws seed + i),
    generated outside every clock."""
    with counter.get_lock():
        idx = counter.value
        counter.value += 1
    _SHARD.update(fmt=fmt, book=book, p=O.Params(fmt, 4, False, chunk, False),
                  words=synth_words(fmt, n, seed + idx, book_w, escapes, rate))


def _step(_):
    s = _SHARD
    t0 = time.perf_counter()
    sec = O.encode(s["words"], s["p"], s["book"])
    t1 = time.perf_counter()
    out = O.decode(sec, s["p"], s["book"])
    t2 = time.perf_counter()
    assert np.array_equal(out, s["words"])
    return s["words"].nbytes, t1 - t0, t2 - t1, int(sec["m"])


class OraclePool:
    """``workers`` processes, one resident shard of ``n_per_worker`` words each."""

    def __init__(self, fmt: int, book, book_w, escapes, rate: float, chunk: int,
                 n_per_worker: int, workers: int, seed: int = 1234):
        self.workers = workers
        self.n_per_worker = n_per_worker
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(workers, initializer=_init,
                             initargs=(ctx.Value("i", 0), fmt, n_per_worker, seed, tuple(book), tuple(book_w),
                                       tuple(escapes), rate, chunk))
        self.pool.map(_noop, range(workers), chunksize=1)  # every shard built

    def step(self, workers: int | None = None) -> dict:
        """One encode + decode of ``workers`` shards (all by default),
        concurrently; GB/s of raw input over the step's wall time."""
        k = self.workers if workers is None else workers
        t0 = time.perf_counter()
        res = self.pool.map(_step, range(k), chunksize=1)
        wall = time.perf_counter() - t0
        total = sum(r[0] for r in res)
        return {"bytes": total, "wall_s": wall, "gbs": total / wall / 1e9,
                "encode_gbs": total / max(r[1] for r in res) / 1e9,
                "decode_gbs": total / max(r[2] for r in res) / 1e9,
                "cpu_seconds": sum(r[1] + r[2] for r in res),
                "escapes": sum(r[3] for r in res)}

    def one_core(self) -> dict:
        """The reference as it runs: one process, one shard."""
        r = self.pool.apply(_step, (0,))
        return {"gbs": r[0] / (r[1] + r[2]) / 1e9, "encode_gbs": r[0] / r[1] / 1e9,
                "decode_gbs": r[0] / r[2] / 1e9, "bytes": r[0]}

    def close(self):
        self.pool.close()
        self.pool.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _noop(_):
    time.sleep(0.01)
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
