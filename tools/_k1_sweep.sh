# K1 TMA knob sweep: builds one library per (input-ring depth, tile-height divisor)
# variant into build/k1var/ (skipped when already built), then times K1 with each
# through tools/bench_stages.py (CUDA-graph replay numbers are the GPU time).
python - <<'PY'
import pathlib, sys
sys.path.insert(0, ".")
from paper_1706_07263_b200 import _build
V = {"s2ty2": (), "s3ty2": ("OXM_K1_STAGES=3",), "s2ty1": ("OXM_K1_TY_DIV=1",), "s2ty4": ("OXM_K1_TY_DIV=4",),
     "s3ty4": ("OXM_K1_STAGES=3", "OXM_K1_TY_DIV=4"), "s4ty4": ("OXM_K1_STAGES=4", "OXM_K1_TY_DIV=4")}
for k, d in V.items():
    out = pathlib.Path(f"build/k1var/{k}/liboximap_b200.so")
    if not out.exists():
        _build.build(force=True, defines=d, out=out)
PY
for v in s2ty2 s3ty2 s2ty1 s2ty4 s3ty4 s4ty4; do
  echo "== $v"
  OXM_LIB_PATH=build/k1var/$v/liboximap_b200.so python tools/bench_stages.py 2>&1 | grep "K1"
done
