#!/usr/bin/env python3
"""Per-kernel SASS instruction mix of the built library (cuobjdump -sass).

    python tools/sass_stats.py [substring] [--top N]
"""

from __future__ import annotations

import collections
import pathlib
import re
import subprocess
import sys

LIB = pathlib.Path(__file__).resolve().parents[1] / "paper_1706_07263_b200" / "_lib" / "liboximap_b200.so"


def kernels() -> dict[str, list[str]]:
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    funcs: dict[str, list[str]] = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if cur and m:
            funcs[cur].append(m.group(2))
    return funcs


def main() -> None:
    sub = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else ""
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    for name, ops in kernels().items():
        if sub not in name:
            continue
        base = collections.Counter(o.split(".")[0] for o in ops)
        print(f"== {name}  ({len(ops)} instructions)")
        print("   " + "  ".join(f"{k}:{v}" for k, v in base.most_common(top)))


if __name__ == "__main__":
    main()
