"""Batched throughput API for video: THb / SO2 maps for many frames per launch.

``HybridMapEngine.run`` is the device-resident path benchmarked as ``value``
(frames already in HBM): eight launches per batch (counter reset, low-pass chain
with the EM start fit, fp32 EM lead-in, fp64 EM tail, fused per-pixel map, fp64
fixup of the flagged pixels with an all-fp64 EM of the few blocks it needs).  ``HybridMapEngine.maps_from_host`` is the end-to-end path
(``e2e``): pinned host frames -> H2D -> kernels -> D2H of the maps, chunked
over three streams so copies in both directions overlap the compute.

Semantics are those of estimate_frame(mode="hybrid") followed by
ConcentrationMap.thb / .sat_o2 (pipeline.py:176-217, core.py:197-209) on the
same (fp32-representable) frames.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .core import CameraSensitivity, ChromophoreBasis, check_grids
from .device import ptr, require_cuda, stream_handle
from .errors import ArgumentError
from .haar import level_dims
from .operators import DEFAULT_FALLBACK_BELOW, DeviceContext, OperatorSet, context
from .pipeline import PipelineConfig, _hybrid_operators


# oxm_ctx_create's default EM schedule (abi.cu): fp32 fits while rel > 16 tol,
# 1% guard band, exact re-estimate of blocks with fallback pixels
DEFAULT_EM_LEAD = (16.0, 0.01)


def _event_array(events):
    """6 torch.cuda.Event -> (void*)[6] of their cudaEvent_t handles."""
    if events is None:
        return None
    import ctypes

    handles = []
    for ev in events:
        if ev.cuda_event == 0:  # created lazily by torch: force creation
            ev.record()
        handles.append(ev.cuda_event)
    if len(handles) != 6:
        raise ArgumentError("stage_events: 6 events (before low-pass, EM lead-in, EM fp64, per-pixel, fixup; after)")
    return (ctypes.c_void_p * 6)(*handles)


@dataclass
class MapBatch:
    thb: torch.Tensor
    so2: torch.Tensor
    hbo: torch.Tensor | None = None
    hb: torch.Tensor | None = None
    offset: torch.Tensor | None = None
    fits: torch.Tensor | None = None
    flags: torch.Tensor | None = None


class HybridMapEngine:
    """Hybrid estimator for (B, H, W, 3) float32 frame batches on one GPU."""

    # zero_counters, ll_tma_kernel (+ EM fit #1), em_lead_kernel, em_persistent_kernel (tail),
    # px_f32_kernel (+ in-warp fp64 fallback), exact pass (em_persistent / em_exact), px_fallback_kernel (deferred)
    KERNELS_PER_RUN = 7

    def __init__(
        self,
        sensitivity: CameraSensitivity,
        basis: ChromophoreBasis,
        cfg: PipelineConfig | None = None,
        *,
        device: torch.device | None = None,
        fallback_below: float = DEFAULT_FALLBACK_BELOW,
        em_lead: tuple | None = DEFAULT_EM_LEAD,
    ):
        """``em_lead``: (ratio, guard[, exact_below[, first_guard[, halvings]]]) of the EM's fp32
        lead-in (oxm_ctx_set_em_lead: fp32 fits while rel > ratio * rel_tol, then
        fp64; fp64 redo of coefficients whose stop decision lands within
        ``guard`` of rel_tol; all-fp64 re-estimate of blocks holding a fallback
        pixel with a band below ``exact_below``, default ``fallback_below``;
        oxm_ctx_set_em_first_guard: guard bands of the tail's first steps), or
        None for all-fp64 EM fits."""
        check_grids(sensitivity.grid, basis.grid)
        self.cfg = cfg if cfg is not None else PipelineConfig(mode="hybrid", n_levels=2)
        if self.cfg.mode != "hybrid":
            raise ArgumentError("HybridMapEngine runs mode='hybrid'")
        self.device = device if device is not None else require_cuda()
        base = _hybrid_operators(sensitivity, basis, self.cfg)
        self.ops = OperatorSet(**{**base.__dict__, "fallback_below": float(fallback_below)})
        self._lib = _native.load()
        if em_lead == DEFAULT_EM_LEAD:
            self.ctx = context(self.ops, self.device.index)
        else:  # a private context: the cached one is shared
            self.ctx = DeviceContext(self.ops, self.device.index)
            lead = tuple(em_lead) if em_lead is not None else (0.0, DEFAULT_EM_LEAD[1])
            ratio, guard = lead[:2]
            exact = lead[2] if len(lead) > 2 else float(fallback_below)
            _native.check(self._lib.oxm_ctx_set_em_lead(self.ctx.handle, float(ratio), float(guard), float(exact)),
                          "em_lead")
            if len(lead) > 3:
                shift = int(lead[4]) if len(lead) > 4 else 2
                _native.check(self._lib.oxm_ctx_set_em_first_guard(self.ctx.handle, float(lead[3]), shift),
                              "em_first_guard")
        self.em_lead = em_lead
        self._ws: torch.Tensor | None = None
        self._audit_args = (sensitivity, basis, float(fallback_below))
        self._audit_engine: HybridMapEngine | None = None

    # ---- workspace ---------------------------------------------------------
    def workspace_bytes(self, batch: int, height: int, width: int) -> int:
        return int(self._lib.oxm_hybrid_workspace_bytes(self.ctx.handle, batch, height, width, self.cfg.n_levels))

    def _workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._ws

    def allocate(self, batch: int, height: int, width: int, *, planes: bool = False, fits: bool = False) -> MapBatch:
        shape = (batch, height, width)
        kw = dict(dtype=torch.float32, device=self.device)
        hL, wL = level_dims(height, width, self.cfg.n_levels)[-1]
        return MapBatch(
            thb=torch.empty(shape, **kw),
            so2=torch.empty(shape, **kw),
            hbo=torch.empty(shape, **kw) if planes else None,
            hb=torch.empty(shape, **kw) if planes else None,
            offset=torch.empty(shape, **kw) if planes else None,
            fits=torch.empty((batch, hL, wL), dtype=torch.int32, device=self.device) if fits else None,
            flags=torch.zeros(1, dtype=torch.int32, device=self.device),
        )

    def em_counters(self, batch: int, height: int, width: int) -> dict:
        """EM work of the last launch of this geometry: fp32 lead-in fits,
        fp64 tail fits, exact-mode restarts, blocks re-estimated all-fp64 for
        the pixel fallback, pixels that took the fp64 fallback and, of those,
        the ones deferred to after the exact pass (synchronises the current
        stream)."""
        import ctypes

        out = (ctypes.c_uint64 * 6)()
        st = self._lib.oxm_hybrid_em_counters(self.ctx.handle, ptr(self._workspace(self.workspace_bytes(batch, height, width))),
                                              batch, height, width, self.cfg.n_levels, out,
                                              stream_handle(None))
        _native.check(st, "em_counters")
        return {"lead_fits": int(out[0]), "tail_fits": int(out[1]), "restarts": int(out[2]),
                "exact_blocks": int(out[3]), "queued_px": int(out[4]), "deferred_px": int(out[5])}

    def audit(self, frames: torch.Tensor, out: MapBatch) -> dict:
        """Runtime check of the EM precision schedule on a batch this engine
        has mapped: ``frames`` again through an all-fp64 EM engine (em_lead=None,
        same operators and configuration; created on first use and kept), then
        every low-pass coefficient's fit count (``out`` must come from
        ``launch`` / ``run`` with ``fits=True``) and the maps compared.  Fit
        counts equal the reference's exactly when this reports 0 flips (the
        all-fp64 schedule is pinned to the oracle by the GPU tests).  Costs one
        all-fp64 run of the batch; synchronises."""
        if out.fits is None:
            raise ArgumentError("audit needs the fit counts: allocate / run with fits=True")
        if self._audit_engine is None:
            sens, basis, fb = self._audit_args
            self._audit_engine = HybridMapEngine(sens, basis, self.cfg, device=self.device, fallback_below=fb,
                                                 em_lead=None)
        ref = self._audit_engine.run(frames, fits=True)
        torch.cuda.synchronize(self.device)
        flips = int((ref.fits != out.fits).sum().item())
        rt = ref.thb.double()
        nz = rt != 0
        thb_rel = float(((out.thb.double() - rt).abs()[nz] / rt.abs()[nz]).max().item()) if bool(nz.any()) else 0.0
        ok = ~torch.isnan(ref.so2)
        so2_abs = float((out.so2[ok] - ref.so2[ok]).abs().max().item()) if bool(ok.any()) else 0.0
        return {"coefficients": int(out.fits.numel()), "fit_count_flips": flips, "max_thb_rel": thb_rel,
                "max_so2_abs": so2_abs,
                "so2_nan_pattern_equal": bool(torch.equal(torch.isnan(out.so2), torch.isnan(ref.so2)))}

    # ---- device-resident path ---------------------------------------------
    def launch(self, frames: torch.Tensor, out: MapBatch, *, stream: torch.cuda.Stream | None = None,
               stage_events=None, scale: float = 1.0, big_endian: bool = True) -> None:
        """Enqueue the hybrid kernels on ``stream``; no host synchronisation.

        The engine owns one workspace (intermediates and the EM / fallback
        counters): launches on different streams must not overlap in time --
        use one engine per concurrent stream.

        ``frames``: CUDA (B, H, W, 3) float32 values, or uint16 PPM counts
        (sample = count * ``scale``; ``big_endian`` as stored in the file).

        Data errors (non-finite samples, negative low-pass) only set bits in
        ``out.flags``: call ``check_flags(out)`` once the stream has finished
        (``run`` and ``maps_from_host`` do) -- the maps of a launch with flags
        set are not the reference's (it raises instead of returning them)."""
        if frames.dim() != 4 or frames.shape[-1] != 3 or not frames.is_cuda:
            raise ArgumentError("frames must be a CUDA (B, H, W, 3) tensor")
        if frames.dtype not in (torch.float32, torch.uint16):
            raise ArgumentError("frames must be float32 values or uint16 PPM counts")
        if not frames.is_contiguous():
            raise ArgumentError("frames must be contiguous")
        B, H, W, _ = frames.shape
        n = self.cfg.n_levels
        if H < 2**n or W < 2**n:
            raise ArgumentError(f"frame {H}x{W} is smaller than 2^{n} in one dimension")
        nbytes = self.workspace_bytes(B, H, W)
        ws = self._workspace(nbytes)
        tail = (B, H, W, n, float(self.cfg.calibration_scale), ptr(ws), nbytes, ptr(out.thb), ptr(out.so2),
                ptr(out.hbo), ptr(out.hb), ptr(out.offset), ptr(out.fits), ptr(out.flags), stream_handle(stream),
                _event_array(stage_events))
        if frames.dtype == torch.float32:
            st = self._lib.oxm_hybrid_maps_f32(self.ctx.handle, ptr(frames), *tail)
        else:
            st = self._lib.oxm_hybrid_maps_u16(self.ctx.handle, ptr(frames), int(big_endian), float(scale), *tail)
        _native.check(st, "hybrid_maps")

    def launch_overlapped(self, frames: torch.Tensor, out: MapBatch, *, parts: int = 4, em_reserve: int = 1,
                          _state: dict | None = None) -> None:
        """Device-resident path with sub-batch pipelining: the per-pixel stage
        of part k (MUFU/FMA) runs on a second stream concurrently with the EM of
        part k+1 (fp64).  Two workspaces alternate between parts.  Ends with
        the current stream waiting for both streams (no host sync)."""
        if frames.dtype != torch.float32 or frames.dim() != 4 or not frames.is_cuda or not frames.is_contiguous():
            raise ArgumentError("frames must be a contiguous CUDA float32 (B, H, W, 3) tensor")
        B, H, W, _ = frames.shape
        n = self.cfg.n_levels
        if H < 2**n or W < 2**n:
            raise ArgumentError(f"frame {H}x{W} is smaller than 2^{n} in one dimension")
        st = _state if _state is not None else {}
        per = -(-B // parts)
        nbytes = self.workspace_bytes(per, H, W)
        if st.get("key") != (per, H, W):
            st.clear()
            st["key"] = (per, H, W)
            st["ws"] = [torch.empty(nbytes, dtype=torch.uint8, device=self.device) for _ in range(2)]
            st["s_em"] = torch.cuda.Stream(device=self.device)
            st["s_px"] = torch.cuda.Stream(device=self.device)
        s_em, s_px, ws = st["s_em"], st["s_px"], st["ws"]
        cur = torch.cuda.current_stream()
        s_em.wait_stream(cur)
        s_px.wait_stream(cur)
        px_done: list = []
        for i, b0 in enumerate(range(0, B, per)):
            nb = min(per, B - b0)
            if i >= 2:
                s_em.wait_event(px_done[i - 2])  # workspace i % 2 is free again
            sl = slice(b0, b0 + nb)
            planes = out.hbo is not None
            rc = self._lib.oxm_hybrid_maps_f32_split(
                self.ctx.handle, ptr(frames[sl]), nb, H, W, n, float(self.cfg.calibration_scale), ptr(ws[i & 1]), nbytes,
                ptr(out.thb[sl]), ptr(out.so2[sl]), ptr(out.hbo[sl]) if planes else None,
                ptr(out.hb[sl]) if planes else None, ptr(out.offset[sl]) if planes else None,
                ptr(out.fits[sl]) if out.fits is not None else None, ptr(out.flags), s_em.cuda_stream,
                s_px.cuda_stream, int(em_reserve))
            _native.check(rc, "hybrid_maps_f32_split")
            ev = torch.cuda.Event()
            ev.record(s_px)
            px_done.append(ev)
        cur.wait_stream(s_em)
        cur.wait_stream(s_px)

    def check_flags(self, out: MapBatch) -> None:
        f = int(out.flags.item())
        if f & _native.FLAG_NONFINITE:
            raise ArgumentError("image contains non-finite values")
        if f & _native.FLAG_NEGATIVE_LL:
            raise ArgumentError("low-pass coefficients must be finite and non-negative")

    def run(self, frames: torch.Tensor, *, planes: bool = False, fits: bool = False, check: bool = True,
            scale: float = 1.0, big_endian: bool = True) -> MapBatch:
        B, H, W, _ = frames.shape
        out = self.allocate(B, H, W, planes=planes, fits=fits)
        self.launch(frames, out, scale=scale, big_endian=big_endian)
        if check:
            self.check_flags(out)
        return out

    # ---- end-to-end host path ---------------------------------------------
    def maps_from_host(
        self,
        frames: torch.Tensor,
        thb_out: torch.Tensor,
        so2_out: torch.Tensor,
        *,
        chunk: int = 8,
        _state: dict | None = None,
        scale: float = 1.0,
        big_endian: bool = True,
    ) -> None:
        """Host (pinned) (B, H, W, 3) frames -> host THb / SO2 (B, H, W).

        Frames are float32 values or uint16 PPM counts (value = count * scale).

        Chunks of ``chunk`` frames are pipelined over three streams: H2D of
        chunk i+1 and D2H of chunk i-1 overlap the kernels of chunk i.  Blocks
        until the last map has landed in host memory, then raises on flags.
        """
        if frames.is_cuda or thb_out.is_cuda or so2_out.is_cuda:
            raise ArgumentError("maps_from_host takes host tensors")
        B, H, W, _ = frames.shape
        st = _state if _state is not None else {}
        key = (chunk, H, W, frames.dtype)
        if st.get("key") != key:
            dev = self.device
            st.clear()
            st["key"] = key
            st["h2d"] = torch.cuda.Stream(device=dev)
            st["comp"] = torch.cuda.Stream(device=dev)
            st["d2h"] = torch.cuda.Stream(device=dev)
            st["in"] = [torch.empty((chunk, H, W, 3), dtype=frames.dtype, device=dev) for _ in range(2)]
            st["out"] = [self.allocate(chunk, H, W) for _ in range(2)]
            st["flags"] = torch.zeros(1, dtype=torch.int32, device=dev)
        h2d, comp, d2h = st["h2d"], st["comp"], st["d2h"]
        ins, outs, flags = st["in"], st["out"], st["flags"]
        flags.zero_()
        loaded = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [None, None]
        consumed = [None, None]
        cur = torch.cuda.current_stream()
        h2d.wait_stream(cur)
        comp.wait_stream(cur)
        d2h.wait_stream(cur)
        for i, b0 in enumerate(range(0, B, chunk)):
            k = i & 1
            nb = min(chunk, B - b0)
            with torch.cuda.stream(h2d):
                if consumed[k] is not None:
                    h2d.wait_event(consumed[k])
                ins[k][:nb].copy_(frames[b0 : b0 + nb], non_blocking=True)
                loaded[k].record(h2d)
            with torch.cuda.stream(comp):
                comp.wait_event(loaded[k])
                if drained[k] is not None:
                    comp.wait_event(drained[k])
                o = outs[k]
                o.flags = flags
                view = MapBatch(thb=o.thb[:nb], so2=o.so2[:nb], flags=flags)
                self.launch(ins[k][:nb], view, stream=comp, scale=scale, big_endian=big_endian)
                ev = torch.cuda.Event()
                ev.record(comp)
                consumed[k] = ev
                computed[k].record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(computed[k])
                thb_out[b0 : b0 + nb].copy_(outs[k].thb[:nb], non_blocking=True)
                so2_out[b0 : b0 + nb].copy_(outs[k].so2[:nb], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(d2h)
                drained[k] = ev
        d2h.synchronize()
        comp.synchronize()
        f = int(flags.item())
        if f & _native.FLAG_NONFINITE:
            raise ArgumentError("image contains non-finite values")
        if f & _native.FLAG_NEGATIVE_LL:
            raise ArgumentError("low-pass coefficients must be finite and non-negative")


def estimate_maps(
    frames: np.ndarray,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    cfg: PipelineConfig | None = None,
    *,
    chunk: int = 8,
) -> tuple[np.ndarray, np.ndarray]:
    """Convenience: NumPy (B, H, W, 3) frames -> (THb, SO2) float32 NumPy maps
    through the pipelined host path."""
    eng = HybridMapEngine(sensitivity, basis, cfg)
    arr = np.ascontiguousarray(frames, dtype=np.float32)
    if arr.ndim == 3:
        arr = arr[None]
    src = torch.from_numpy(arr).pin_memory()
    B, H, W, _ = arr.shape
    thb = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
    so2 = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
    eng.maps_from_host(src, thb, so2, chunk=chunk)
    return thb.numpy().copy(), so2.numpy().copy()
