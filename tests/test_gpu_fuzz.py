"""Randomised parity against the oracle (a short run of tools/parity_fuzz.py:
random odd/even sizes, 1-4 levels, batches, texture and exposure; fp32 engine
with bit-exact fit counts and the fp64 drop-in)."""

from __future__ import annotations

import json

import pytest

pytestmark = pytest.mark.gpu


def test_randomised_parity(cuda):
    from tools import parity_fuzz

    lines = []
    summary = parity_fuzz.run(12, 7, emit=lines.append)
    bad = [json.loads(x) for x in lines if '"pass": false' in x]
    assert summary["failed"] == 0, bad
