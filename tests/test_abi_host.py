"""CPU-side checks of the C ABI library and the host logic (no kernels run)."""

from __future__ import annotations

import ctypes
import re

import numpy as np
import pytest

from paper_1706_07263_b200 import _native


def _header_functions() -> set[str]:
    text = _native.HEADER_PATH.read_text()
    return set(re.findall(r"OXM_API\s+[\w\s\*]+?\b(oxm_\w+)\s*\(", text))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    declared = _header_functions()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes table binds exactly the header's functions
    assert set(_native.exported_names()) == declared


def test_abi_version_and_status_strings():
    lib = _native.load()
    assert lib.oxm_abi_version() == 2
    for code, text in [(0, b"ok"), (-1, b"argument error"), (-2, b"data error"), (-10, b"cuda error")]:
        assert lib.oxm_status_string(code) == text


def test_haar_layout_host_only():
    lib = _native.load()
    hw = (ctypes.c_int64 * 6)()
    tot = ctypes.c_int64()
    assert lib.oxm_haar_layout(1080, 1920, 3, ctypes.addressof(hw), ctypes.addressof(tot)) == 0
    assert list(hw) == [540, 960, 270, 480, 135, 240]
    assert tot.value == 4 * (540 * 960 + 270 * 480 + 135 * 240)
    assert lib.oxm_haar_layout(9, 15, 1, ctypes.addressof(hw), None) == 0
    assert list(hw)[:2] == [5, 8]
    assert lib.oxm_haar_layout(0, 4, 1, None, None) == _native.OXM_ERR_ARGUMENT
    assert lib.oxm_haar_layout(4, 4, 0, None, None) == _native.OXM_ERR_ARGUMENT


def test_status_mapping_to_reference_exceptions():
    from paper_1706_07263_b200.errors import (
        ArgumentError,
        DataError,
        IllConditionedPriorError,
        NativeLibraryError,
        NumericalError,
        SingularOperatorError,
    )

    for code, cls in [(-1, ArgumentError), (-2, DataError), (-3, NumericalError), (-4, SingularOperatorError),
                      (-5, IllConditionedPriorError), (-10, NativeLibraryError)]:
        with pytest.raises(cls):
            _native.check(code, "x")
    assert issubclass(ArgumentError, ValueError)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1706_07263_b200 import NativeLibraryError, PipelineConfig, RgbImage, estimate_frame, fixtures, forward

    with pytest.raises(NativeLibraryError):
        forward(np.ones((4, 4)), 1)
    with pytest.raises(NativeLibraryError):
        estimate_frame(RgbImage(np.ones((8, 8, 3))), fixtures.default_sensitivity(), fixtures.default_basis(),
                       PipelineConfig(n_levels=1))


def test_fixtures_match_reference_tables(golden, sensitivity, basis):
    from paper_1706_07263_b200 import WavelengthGrid, fixtures

    g = golden("operators")
    assert np.array_equal(sensitivity.c, g["c"])
    assert np.array_equal(basis.xi, g["xi"])
    g55 = WavelengthGrid(440.0, 5.0, 55)
    assert np.array_equal(fixtures.default_sensitivity(g55).c, g["c55"])
    assert np.array_equal(fixtures.default_basis(g55).xi, g["xi55"])


def test_synth_reproduces_reference_phantoms(golden, sensitivity, basis):
    from paper_1706_07263_b200 import synth

    g = golden("frames")
    seeds_td = {0: (1, 0.3), 1: (2, 0.3), 2: (3, 0.3), 3: (4, 0.0), 5: (6, 0.3)}
    for i, (seed, td) in seeds_td.items():
        H, W = (int(v) for v in g[f"meta{i}"][:2])
        got = synth.phantom_rgb_f32(H, W, seed, sensitivity, basis, texture_density=td)
        assert np.array_equal(got, g[f"rgb{i}"]), i


def test_host_operators(sensitivity, basis, golden):
    from paper_1706_07263_b200 import TikhonovOperator
    from paper_1706_07263_b200.operators import ShapePrior, fit_matrix

    op = TikhonovOperator.from_relative(sensitivity, 1e-3)
    assert np.array_equal(op.solve, golden("operators")["solve"])
    prior = ShapePrior.build(sensitivity.c, 0.1)
    # G = N^-1 C^T and the identity N^-1 P = I - G C used by the kernels
    N = sensitivity.c.T @ sensitivity.c + prior.prior
    assert np.allclose(N @ prior.gain, sensitivity.c.T, atol=1e-12)
    lhs = np.linalg.solve(N, prior.prior)
    assert np.allclose(lhs, np.eye(26) - prior.gain @ sensitivity.c, atol=1e-9)
    F = fit_matrix(basis.xi)
    assert np.allclose(F @ basis.xi, np.eye(3), atol=1e-12)


class TestValidation:
    def test_configs(self):
        from paper_1706_07263_b200 import ArgumentError, BayesConfig, PipelineConfig

        for kw in [dict(beta=0.0), dict(max_iters=0), dict(rel_tol=0.0), dict(epsilon=0.0), dict(epsilon=1.0)]:
            with pytest.raises(ArgumentError):
                BayesConfig(**kw)
        for kw in [dict(mode="magic"), dict(n_levels=0), dict(tikhonov_gamma=0.0), dict(threads=0),
                   dict(calibration_scale=0.0)]:
            with pytest.raises(ArgumentError):
                PipelineConfig(**kw)

    def test_lowpass_block_rejects_negative(self):
        from paper_1706_07263_b200 import ArgumentError, LowPassBlock

        with pytest.raises(ArgumentError):
            LowPassBlock(rgb_lp=np.full((2, 2, 3), -0.5), scale=1.0)
        with pytest.raises(ArgumentError):
            LowPassBlock(rgb_lp=np.ones((2, 2, 3)), scale=0.0)

    def test_gamma_positive(self, sensitivity):
        from paper_1706_07263_b200 import ArgumentError, TikhonovOperator

        with pytest.raises(ArgumentError):
            TikhonovOperator.build(sensitivity, 0.0)

    def test_ill_conditioned_prior(self):
        from paper_1706_07263_b200 import CameraSensitivity, IllConditionedPriorError, WavelengthGrid
        from paper_1706_07263_b200.operators import ShapePrior

        # rows symmetric about the centre band: the centred ramp lies in
        # null(C) and in null(D2), so N = C^T C + beta D2^T D2 is singular
        L = 9
        t = np.arange(L) - (L - 1) / 2
        rows = np.stack([np.exp(-0.5 * (t / s) ** 2) for s in (1.0, 2.0, 4.0)])
        sens = CameraSensitivity(WavelengthGrid(500.0, 10.0, L), rows)
        with pytest.raises(IllConditionedPriorError):
            ShapePrior.build(sens.c, 0.1)

    def test_pyramid_shape_errors(self):
        from paper_1706_07263_b200 import ArgumentError, DataError, HaarLevel, HaarPyramid
        from paper_1706_07263_b200.haar import _check_chain

        lv = HaarLevel(lp=np.zeros((4, 4)), dh=np.zeros((2, 4)), dv=np.zeros((4, 4)), dd=np.zeros((4, 4)),
                       orig_shape=(8, 8))
        with pytest.raises(DataError):
            _check_chain(HaarPyramid(levels=(lv,)))
        with pytest.raises(ArgumentError):
            HaarPyramid(levels=())
        with pytest.raises(ArgumentError):
            HaarPyramid(levels=(HaarLevel(lp=None, dh=np.zeros((2, 2)), dv=np.zeros((2, 2)), dd=np.zeros((2, 2)),
                                          orig_shape=(4, 4)),))
        ok = HaarLevel(lp=np.zeros((3, 5, 2)), dh=np.zeros((3, 5, 2)), dv=np.zeros((3, 5, 2)),
                       dd=np.zeros((3, 5, 2)), orig_shape=(5, 9))
        assert _check_chain(HaarPyramid(levels=(ok,))) == [(3, 5, 5, 9)]

    def test_core_types(self):
        from paper_1706_07263_b200 import (
            ArgumentError,
            ConcentrationMap,
            DataError,
            RgbImage,
            SpectralCube,
            WavelengthGrid,
            check_grids,
        )

        with pytest.raises(ArgumentError):
            RgbImage(np.full((2, 2, 3), np.inf))
        with pytest.raises(ArgumentError):
            RgbImage(np.ones((2, 2, 4)))
        with pytest.raises(DataError):
            SpectralCube(WavelengthGrid(450, 10, 26), np.ones((2, 2, 25)))
        with pytest.raises(DataError):
            check_grids(WavelengthGrid(450, 10, 26), WavelengthGrid(450, 10, 27))
        m = ConcentrationMap(hbo=np.array([[1.0, -1.0, 0.0]]), hb=np.array([[1.0, 2.0, -3.0]]),
                             offset=np.zeros((1, 3)))
        assert np.array_equal(m.thb, [[2.0, 2.0, 0.0]])
        assert np.array_equal(m.sat_o2, [[0.5, 0.0, np.nan]], equal_nan=True)


class TestPpmHeader:
    """read_ppm_raw follows the reference header grammar (io.py:112-162)."""

    def _write(self, tmp_path, header: bytes, raster: bytes):
        p = tmp_path / "f.ppm"
        p.write_bytes(header + raster)
        return p

    def test_roundtrip_and_scale(self, tmp_path):
        from paper_1706_07263_b200.io import read_ppm_raw

        counts = np.arange(2 * 3 * 3, dtype=">u2").reshape(2, 3, 3)
        p = self._write(tmp_path, b"P6\n# scale 0.5\n3 2\n65535\n", counts.tobytes())
        raw, scale = read_ppm_raw(p)
        assert scale == 0.5
        assert np.array_equal(raw.view(">u2"), counts)  # file byte order, decoded on device
        p2 = self._write(tmp_path, b"P6 3 2 65535\n", counts.tobytes())
        assert read_ppm_raw(p2)[1] == 1.0

    @pytest.mark.parametrize("header,raster", [
        (b"P5\n3 2\n65535\n", b"\0" * 36),
        (b"P6\n3 2\n255\n", b"\0" * 36),
        (b"P6\n3 2\n65535\n", b"\0" * 35),
        (b"P6\n# scale nope\n3 2\n65535\n", b"\0" * 36),
        (b"P6\n3", b""),
    ])
    def test_malformed(self, tmp_path, header, raster):
        from paper_1706_07263_b200 import DataError
        from paper_1706_07263_b200.io import read_ppm_raw

        with pytest.raises(DataError):
            read_ppm_raw(self._write(tmp_path, header, raster))
