"""The reference's container-robustness harnesses through the GPU decode
path: every mutated container of tests/golden/robust.* (truncation at every
offset, 1500 bit flips with seed 2024, 1000 byte XORs with seed 1234, every
pad bit, and the same harness over the E5M2 / E4M3 / sentinel / abs32 /
3-bit bases) goes through ``decode_container`` twice — as host bytes and as
a CUDA uint8 tensor (sections sliced in HBM, K3 + K4 validate) — and must
end exactly as the reference did (pkg/tests/test_container.py:134-165,
pkg/tests/test_acceptance.py:295-337):

* rejected while parsing or decoding: same exception class, ``section``,
  ``chunk`` and message;
* decoded: the same words as the reference's decode of the damaged bytes
  (BLAKE2b digest), never a CUDA error and never a silent success the
  reference did not also have."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from sz_testutil import robust, words_digest

pytestmark = pytest.mark.gpu


def _bases():
    return sorted(robust().bases)


def _outcome(fn, data):
    import paper_2605_01708_b200 as m
    try:
        dec = fn(data)
    except m.SplitZipError as exc:
        return ("raise", type(exc).__name__, getattr(exc, "section", None),
                getattr(exc, "chunk", None), str(exc))
    w = dec.words
    w = w.cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w)
    return ("ok", words_digest(w), int(w.size))


def _want(v):
    if v["stage"] == "ok":
        return ("ok", v["digest"], v["n"])
    return ("raise", v["raised"], v["section"], v["chunk"], v["msg"])


@pytest.mark.parametrize("path", ["auto", "k3e"])
@pytest.mark.parametrize("where", ["host", "device"])
@pytest.mark.parametrize("bid", _bases())
def test_decode_container_verdicts_match_reference(bid, where, path, monkeypatch):
    # "k3e": every chunk-relative decode (chunk >= 32) forced through the
    # escape-dense pre-pass path, whatever its escape rate
    if path == "k3e":
        monkeypatch.setenv("SZ_DEC_MARKED", "1")
    from paper_2605_01708_b200.container import decode_container
    r = robust()
    bad = []
    for v in (v for v in r.verdicts if v["base"] == bid):
        data = r.mutated(v)
        if where == "device":
            data = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda() if data else \
                torch.empty(0, dtype=torch.uint8, device="cuda")
        got = _outcome(decode_container, data)
        if got != _want(v):
            bad.append((v["kind"], v["mut"], _want(v), got))
    torch.cuda.synchronize()   # a device fault surfaces here, not as a verdict
    assert not bad, f"{len(bad)} verdicts differ, e.g. {bad[:4]}"
