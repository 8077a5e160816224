"""Real-KV golden fixtures, produced by running the REAL reference packages.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_realkv.py

1. Runs ``kv_extractor.extract`` exactly as the reference's interop tests do
   (``pkg/kv_extractor/tests/test_extract.py:84-88``: the offline
   ``random-gpt2`` target of ``extract.py:85-94``, SAMPLE_PROMPTS,
   ``max_tokens=128``, seed 0).  Its dumps are real attention K/V
   activations in the ``.szrw`` layout (``extract.py:66-72``): 4 layers x
   {K, V} BF16 files.
2. Derives FP8 E5M2 dumps from the same activations by the cast an FP8 KV
   cache applies on write (``tensor.to(torch.float8_e5m2)``), so config 3's
   format also has real-activation parity data.
3. Runs the reference ``splitzip`` on them and records what its CLI
   ``calibrate`` (cli.py:164-199: per-file ``build_histogram``,
   ``merge_stats``, ``entropy_bits``, top-8/16 coverage, ``select_codebook``,
   ``coverage_by_group``) and ``verify --dynamic`` / ``compress`` (cli.py:
   214-228, 254-...) produce: per dump and codec config, the SHA-256 of every
   payload section, M, ``payload_nbytes`` and the container file's SHA-256.

Output, committed: ``tests/golden/realkv/*.szrw`` (the BF16 dumps, byte for
byte what kv_extractor wrote, + manifest.json) and
``tests/golden/realkv.json`` (reference results).  The E5M2 dumps are not
stored; tests rebuild them from the BF16 words with torch's cast and check
them against the SHA-256 recorded here.  Nothing on the GPU box reads
``/root/reference``.
"""

from __future__ import annotations

import hashlib
import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "realkv"

# (name, code_bits, mode, chunk, position_mode, shared-calibrated book?)
CONFIGS = [
    ("dyn4", 4, "explicit", 1024, "chunk", False),   # verify --dynamic
    ("cal4", 4, "explicit", 1024, "chunk", True),    # calibrate -> compress
    ("cal4_c256", 4, "explicit", 256, "chunk", True),
    ("cal3", 3, "explicit", 1024, "chunk", True),
    ("cal4_sent", 4, "sentinel", 1024, "chunk", True),
    ("cal4_abs32", 4, "explicit", 1024, "abs32", True),
]


def load_reference():
    scratch = Path(tempfile.mkdtemp(prefix="szref_"))
    shutil.copytree("/root/reference/pkg/src/splitzip", scratch / "splitzip")
    shutil.copytree("/root/reference/pkg/kv_extractor/src/kv_extractor",
                    scratch / "kv_extractor")
    sys.path.insert(0, str(scratch))
    import importlib
    import splitzip  # noqa: E402
    # kv_extractor/__init__ re-exports the function ``extract``, which shadows
    # the submodule attribute; fetch the module itself.
    kx = importlib.import_module("kv_extractor.extract")
    return splitzip, kx


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(bytes(b)).hexdigest()


def e5m2_words(bf16_words: np.ndarray) -> np.ndarray:
    import torch
    t = torch.from_numpy(bf16_words.astype(np.uint16).view(np.int16)).view(torch.bfloat16)
    return t.to(torch.float8_e5m2).view(torch.uint8).numpy().copy()


def main():
    sz, kx = load_reference()
    from splitzip import container as C
    from splitzip.calibration import (build_histogram, coverage_by_group, entropy_bits,
                                      merge_stats, select_codebook, top_k_coverage)

    if OUT.exists():
        shutil.rmtree(OUT)
    manifest = kx.extract("random-gpt2", kx.SAMPLE_PROMPTS, 128, OUT, seed=0)

    result = {"extract": {"model": "random-gpt2", "prompts": "SAMPLE_PROMPTS",
                          "max_tokens": 128, "seed": 0, "manifest": manifest},
              "formats": {}}
    files = [OUT / r["path"] for r in manifest["files"]]
    bf16_streams = [C.read_raw_tensor(p) for p in files]
    e5_streams = [sz.RawTensorStream(sz.ElementFormat.FP8_E5M2, e5m2_words(s.words))
                  for s in bf16_streams]

    for fname, streams in (("bf16", bf16_streams), ("e5m2", e5_streams)):
        fmt = streams[0].fmt
        parts = [build_histogram(s) for s in streams]
        stats = merge_stats(*parts)
        books = {}
        for cb, mode in ((4, "explicit"), (3, "explicit"), (4, "sentinel")):
            books[(cb, mode)] = select_codebook(stats, cb, sz.CodebookMode.from_name(mode))
        fres = {
            "calibrate": {
                "elements": int(stats.total),
                "counts": [int(c) for c in stats.counts],
                "entropy_bits": float(entropy_bits(stats)),
                "top8_coverage": float(top_k_coverage(stats, min(8, fmt.exp_bins))),
                "top16_coverage": float(top_k_coverage(stats, min(16, fmt.exp_bins))),
                "books": {f"{cb}_{mode}": list(map(int, b.entries))
                          for (cb, mode), b in books.items()},
                "codebook_record_sha256": sha(C.codebook_record_bytes(books[(4, "explicit")])),
                "group_coverage_1024": [
                    [float(x) for x in coverage_by_group(s, 1024, books[(4, "explicit")])]
                    for s in streams],
            },
            "dumps": [],
        }
        for path, s in zip(files, streams):
            d = {"file": path.name, "n": int(s.n_elements),
                 "words_sha256": sha(s.words), "configs": {}}
            for name, cb, mode, chunk, pos, shared in CONFIGS:
                cfg = sz.CodecConfig(
                    fmt, cb, sz.CodebookMode.from_name(mode), chunk_size=chunk,
                    position_mode=sz.PositionMode.validate(pos),
                    codebook=books[(cb, mode)] if shared else None)
                enc = sz.encode(s, cfg)
                dec = sz.decode(enc, cfg, enc.codebook)
                assert np.array_equal(dec.words, s.words)
                cont = C.container_to_bytes(enc, cfg, enc.codebook)
                d["configs"][name] = {
                    "book": list(map(int, enc.codebook.entries)),
                    "m": int(enc.n_escapes),
                    "payload_nbytes": int(enc.payload_nbytes),
                    "sections": {k: sha(v) for k, v in enc.section_bytes()},
                    "container_sha256": sha(cont),
                    "container_nbytes": len(cont),
                }
            fres["dumps"].append(d)
        result["formats"][fname] = fres
        cal = fres["calibrate"]
        print(f"{fname}: {cal['elements']} elements, entropy {cal['entropy_bits']:.2f} "
              f"bits, top-16 coverage {cal['top16_coverage']:.4%}")

    (HERE / "realkv.json").write_text(json.dumps(result, indent=1))
    print(f"wrote {OUT} and {HERE / 'realkv.json'}")


if __name__ == "__main__":
    main()
