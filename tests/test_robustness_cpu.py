"""The reference's container-robustness harnesses on the host parse path
(``container_from_bytes``): truncation at every offset
(pkg/tests/test_container.py:134-138, test_acceptance.py:295-309), 1500
single-bit flips (test_container.py:146-165), 1000 byte XORs
(test_acceptance.py:311-337), every pad bit (codec.py:236-237,255-256,441-442)
and the same harness over E5M2 / E4M3 / sentinel / abs32 / 3-bit bases.

Every mutation the reference rejects while PARSING must be rejected here
with the same class, section, chunk and message; every mutation the
reference parses must parse here too.  The decode stage (GPU kernels) is
checked by tests/test_gpu_robustness.py."""

from __future__ import annotations

from collections import Counter

import pytest

from sz_testutil import robust


def C():
    from paper_2605_01708_b200 import container
    return container


def _bases():
    return sorted(robust().bases)


def test_verdict_count():
    r = robust()
    kinds = Counter(v["kind"] for v in r.verdicts)
    assert kinds["bitflip"] >= 1500 and kinds["bytexor"] >= 1000
    assert sum(n for k, n in kinds.items() if k.startswith("pad_")) > 0
    assert len(r.verdicts) >= 2500


@pytest.mark.parametrize("bid", _bases())
def test_host_parse_verdicts_match_reference(bid):
    import paper_2605_01708_b200 as m
    r = robust()
    bad = []
    for v in (v for v in r.verdicts if v["base"] == bid):
        data = r.mutated(v)
        try:
            C().container_from_bytes(data)
            got = None
        except m.SplitZipError as exc:
            got = (type(exc).__name__, getattr(exc, "section", None),
                   getattr(exc, "chunk", None), str(exc))
        want = ((v["raised"], v["section"], v["chunk"], v["msg"])
                if v["stage"] == "parse" else None)
        if got != want:
            bad.append((v["kind"], v["mut"], want, got))
    assert not bad, f"{len(bad)} parse verdicts differ, e.g. {bad[:5]}"
