"""Test helpers shared by the suites (golden fixtures, oracle params)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = ROOT / "tests" / "golden"



class Golden:
    """Lazy view over tests/golden/{golden.npz,manifest.json}."""

    def __init__(self):
        self.manifest = json.loads((GOLDEN_DIR / "manifest.json").read_text())
        self._npz = np.load(GOLDEN_DIR / "golden.npz")
        self.cases = self.manifest["cases"]
        self.corruptions = self.manifest["corruptions"]
        self.corruption_bases = self.manifest.get("corruption_bases", {})

    def corruption_base(self, verdict: dict):
        """(base descriptor, original words) of a corruption verdict; verdicts
        without a base mutate the BF16 explicit chunk-relative encode whose
        book is the top 16 of its own histogram."""
        bid = verdict.get("base")
        if bid is None:
            return None, self.arr("corrupt", "words")
        return self.corruption_bases[bid], self.arr(f"corrupt_base_{bid}", "words")

    def corruption_sections(self, verdict: dict) -> dict:
        pre = f"corrupt_{verdict['id']}"
        return {
            "n": verdict["n"], "m": verdict["m"],
            "packed_codes": self.arr(pre, "packed_codes").tobytes(),
            "sign_mantissa": self.arr(pre, "sign_mantissa").tobytes(),
            "chunk_counts": self.arr(pre, "chunk_counts"),
            "escape_positions": self.arr(pre, "escape_positions"),
            "escape_values": self.arr(pre, "escape_values"),
        }

    def arr(self, cid: str, name: str) -> np.ndarray:
        return self._npz[f"{cid}/{name}"]

    def case(self, cid: str) -> dict:
        return next(c for c in self.cases if c["id"] == cid)


_GOLDEN = None


def golden() -> Golden:
    global _GOLDEN
    if _GOLDEN is None:
        _GOLDEN = Golden()
    return _GOLDEN


def golden_case_ids(tag: str | None = None):
    return [c["id"] for c in golden().cases if tag is None or c["tag"] == tag]


def oracle_params(case: dict):
    from oracle import sz_oracle as O
    return O.Params(case["fmt"], case["code_bits"], case["sentinel"], case["chunk"],
                    case["abs32"])


class Robust:
    """Lazy view over tests/golden/{robust.npz,robust.json.gz}: the reference's
    verdicts on mutated containers (tests/golden/make_robustness.py)."""

    def __init__(self):
        import gzip
        with gzip.open(GOLDEN_DIR / "robust.json.gz", "rb") as f:
            meta = json.loads(f.read())
        self.bases = meta["bases"]
        self.verdicts = meta["verdicts"]
        self._npz = np.load(GOLDEN_DIR / "robust.npz")
        self._cache: dict[str, tuple[bytes, np.ndarray]] = {}

    def base(self, bid: str) -> tuple[bytes, np.ndarray]:
        if bid not in self._cache:
            self._cache[bid] = (self._npz[f"{bid}/container"].tobytes(),
                                self._npz[f"{bid}/words"])
        return self._cache[bid]

    def mutated(self, v: dict) -> bytes:
        data, _ = self.base(v["base"])
        if v["kind"] == "truncate":
            return data[:v["mut"]]
        pos, x = v["mut"]
        b = bytearray(data)
        b[pos] ^= x
        return bytes(b)


_ROBUST = None


def robust() -> Robust:
    global _ROBUST
    if _ROBUST is None:
        _ROBUST = Robust()
    return _ROBUST


def words_digest(words: np.ndarray) -> str:
    import hashlib
    return hashlib.blake2b(np.ascontiguousarray(words).tobytes(), digest_size=16).hexdigest()


class RealKV:
    """Real attention K/V dumps (kv_extractor's offline random-gpt2,
    tests/golden/make_realkv.py) and the reference's results on them.
    BF16 words come from the committed .szrw files; the E5M2 words are the
    FP8 KV-cache cast of the same activations, rebuilt here and checked
    against the reference's SHA-256."""

    CONFIGS = {  # name -> (code_bits, sentinel, chunk, abs32, shared book key)
        "dyn4": (4, False, 1024, False, None),
        "cal4": (4, False, 1024, False, "4_explicit"),
        "cal4_c256": (4, False, 256, False, "4_explicit"),
        "cal3": (3, False, 1024, False, "3_explicit"),
        "cal4_sent": (4, True, 1024, False, "4_sentinel"),
        "cal4_abs32": (4, False, 1024, True, "4_explicit"),
    }

    def __init__(self):
        self.dir = GOLDEN_DIR / "realkv"
        self.ref = json.loads((GOLDEN_DIR / "realkv.json").read_text())
        self._words: dict[tuple[str, str], np.ndarray] = {}

    def files(self) -> list[str]:
        return [d["file"] for d in self.ref["formats"]["bf16"]["dumps"]]

    def dump(self, fmt: str, file: str) -> dict:
        return next(d for d in self.ref["formats"][fmt]["dumps"] if d["file"] == file)

    def calibrate(self, fmt: str) -> dict:
        return self.ref["formats"][fmt]["calibrate"]

    def words(self, fmt: str, file: str) -> np.ndarray:
        key = (fmt, file)
        if key not in self._words:
            data = (self.dir / file).read_bytes()
            n = int.from_bytes(data[6:14], "little")
            bf16 = np.frombuffer(data, dtype="<u2", count=n, offset=14).copy()
            if fmt == "bf16":
                self._words[key] = bf16
            else:
                import torch
                t = torch.from_numpy(bf16.view(np.int16)).view(torch.bfloat16)
                self._words[key] = t.to(torch.float8_e5m2).view(torch.uint8).numpy().copy()
        return self._words[key]


_REALKV = None


def realkv() -> RealKV:
    global _REALKV
    if _REALKV is None:
        _REALKV = RealKV()
    return _REALKV


def sha256(b) -> str:
    import hashlib
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(bytes(b)).hexdigest()
