#!/usr/bin/env python3
"""profiles/traffic.json from an ncu report of tools/profile_hybrid.py:
DRAM bytes (read + write) per frame for each bench stage.
    python tools/ncu_traffic.py rep.ncu-rep FRAMES_PER_LAUNCH"""
import csv, io, json, pathlib, subprocess, sys

STAGES = {"ll_kernel": ("ll_kernel",), "em_lead": ("em_lead",), "em": ("em_persistent_kernel<26, 1, 1>",),
          "px_f32_kernel": ("px_f32",),
          # the exact-block pass: 4-lane kernel (small batches) or the one-lane persistent kernel
          "fixup": ("px_fallback", "em_exact", "em_persistent_kernel<26, 1, 0>")}


def main():
    rep, frames = sys.argv[1], float(sys.argv[2])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in data:
        name = r[hdr.index("Kernel Name")]
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            b += float(r[i]) * scale[units[i]]
        for stage, keys in STAGES.items():
            if any(key in name for key in keys):
                per.setdefault(stage, {}).setdefault(name.split("(")[0], []).append(b)
    res = {st: sum(sum(v) / len(v) for v in ks.values()) / frames for st, ks in per.items()}
    dst = pathlib.Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
    dst.parent.mkdir(exist_ok=True)
    dst.write_text(json.dumps({"source": rep, "frames_per_launch": frames, "dram_bytes_per_frame": res}, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
