"""The driver's round-end smoke check, as a GPU test: __graft_entry__.smoke()
(one tiny hybrid pass on cuda:0, fp32 engine and fp64 drop-in, against the
oracle)."""

from __future__ import annotations

import pytest


@pytest.mark.gpu
def test_graft_entry_smoke():
    import __graft_entry__

    __graft_entry__.smoke()
