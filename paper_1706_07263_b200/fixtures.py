"""Default camera sensitivity and chromophore basis.

The reference ships these as CSV tables (pkg/src/oximap/data/*.csv) that its
tools/gen_fixtures.py:22-48 synthesises from sums of Gaussians and rounds to
six significant digits.  Rather than vendoring the files, the same published
curve parameters are evaluated here, rounded the same way, and resampled onto
the requested grid exactly like fixtures.py:23-30 -> io.py:192-214.  A CPU
test checks the result bit-for-bit against the reference tables
(tests/golden/operators.npz).
"""

from __future__ import annotations

import numpy as np

from .core import DEFAULT_GRID, CameraSensitivity, ChromophoreBasis, WavelengthGrid, resample_to_grid

# (amplitude, centre nm, sigma nm) per curve; constant terms as (c, None, None)
_CAMERA = {
    "red": ((0.92, 605, 32), (0.015, 460, 40)),
    "green": ((1.00, 540, 34), (0.010, 640, 40)),
    "blue": ((0.90, 462, 26), (0.012, 550, 45)),
}
_ATTENUATION = {
    "hbo": ((0.036, 445, 26), (0.0186, 542, 12), (0.0174, 577, 11), (0.0021, None, None), (0.0009, 700, 90)),
    "hb": ((0.0378, 435, 28), (0.0276, 556, 22), (0.0045, None, None), (0.0036, 757, 55)),
}


def _curve(wl: np.ndarray, terms) -> np.ndarray:
    out = np.zeros_like(wl)
    for amp, centre, sigma in terms:
        if centre is None:
            out = out + amp
        else:
            out = out + amp * np.exp(-0.5 * ((wl - centre) / sigma) ** 2)
    return out


def _six_digits(values: np.ndarray) -> np.ndarray:
    # the tables store '%.6g' text; parse it back the way the CSV loader does
    return np.array([float(f"{v:.6g}") for v in values])


def camera_table() -> tuple[np.ndarray, dict[str, np.ndarray]]:
    wl = np.arange(440.0, 711.0, 5.0)
    return wl, {k: _six_digits(_curve(wl, t)) for k, t in _CAMERA.items()}


def attenuation_table() -> tuple[np.ndarray, dict[str, np.ndarray]]:
    wl = np.arange(440.0, 711.0, 2.0)
    return wl, {k: _six_digits(_curve(wl, t)) for k, t in _ATTENUATION.items()}


def default_sensitivity(grid: WavelengthGrid = DEFAULT_GRID) -> CameraSensitivity:
    wl, cols = camera_table()
    rows = [resample_to_grid(np.column_stack([wl, cols[k]]), grid) for k in ("red", "green", "blue")]
    return CameraSensitivity(grid=grid, c=np.stack(rows))


def default_basis(grid: WavelengthGrid = DEFAULT_GRID) -> ChromophoreBasis:
    wl, cols = attenuation_table()
    cs = [resample_to_grid(np.column_stack([wl, cols[k]]), grid) for k in ("hbo", "hb")]
    return ChromophoreBasis(grid=grid, xi=np.column_stack(cs + [np.ones(grid.count)]))
