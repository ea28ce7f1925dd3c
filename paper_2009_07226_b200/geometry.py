"""Parallel-beam geometry, GPU Siddon system matrix, phantoms, measurements.

Mirrors the reference module ``xct.geometry`` (src/geometry.py) -- same
names, fields, validation and conventions -- with the ray tracing done by
the sm_100a Siddon kernels of ``libxct_b200.so`` (K1/K2).  The matrix is
built on the device (int64 row pointers, int32 voxel ids in traversal order,
float64 lengths); host numpy copies are materialized lazily, only when a
caller reads ``indptr`` / ``indices`` / ``values``.

Conventions (src/geometry.py:4-14): flat voxel id iz*N + ix; ray r =
k*N + c travels along (cos a_k, sin a_k) offset by rho_c = (c-(N-1)/2)*pitch
along (-sin a_k, cos a_k).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["ScanGeometry", "RaySegmentList", "SystemMatrix", "Volume", "make_geometry",
           "trace_ray", "build_system_matrix", "clear_matrix_cache", "build_count",
           "generate_phantom", "simulate_measurements", "PHANTOM_KINDS", "device"]

PHANTOM_KINDS = ("uniform-disk", "shepp-logan-like", "random-blobs")


def device():
    """The CUDA device the product path runs on (raises without one)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2009_07226_b200 runs on a CUDA device (B200); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class ScanGeometry:
    """K angles, M slices, N detector columns (src/geometry.py:43-68)."""

    num_angles: int
    angles: tuple
    num_rows: int
    num_detector_cols: int
    voxel_size: float = 1.0

    @property
    def grid_n(self) -> int:
        return self.num_detector_cols

    @property
    def detector_pitch(self) -> float:
        return self.voxel_size

    @property
    def num_rays(self) -> int:
        return self.num_angles * self.num_detector_cols

    @property
    def num_voxels(self) -> int:
        return self.grid_n * self.grid_n


def make_geometry(num_angles: int, num_rows: int, num_detector_cols: int,
                  angle_start: float = 0.0, angle_end: float = math.pi,
                  voxel_size: float = 1.0) -> ScanGeometry:
    """Equally spaced views in [angle_start, angle_end) (src/geometry.py:71-87)."""
    if num_angles < 1 or num_rows < 1 or num_detector_cols < 1:
        raise ValueError("K, M and N must all be >= 1")
    if not angle_start < angle_end:
        raise ValueError(f"inverted angle range [{angle_start}, {angle_end})")
    if angle_end - angle_start > math.pi + 1e-12:
        raise ValueError("angle range wider than pi is redundant for parallel beams")
    if voxel_size <= 0:
        raise ValueError("voxel_size must be positive")
    step = (angle_end - angle_start) / num_angles
    return ScanGeometry(num_angles=num_angles,
                        angles=tuple(angle_start + i * step for i in range(num_angles)),
                        num_rows=num_rows, num_detector_cols=num_detector_cols,
                        voxel_size=voxel_size)


@dataclass(frozen=True)
class RaySegmentList:
    """Ordered (voxel id, length) pairs of one ray (src/geometry.py:90-105)."""

    indices: np.ndarray = field(repr=False)
    lengths: np.ndarray = field(repr=False)

    def __len__(self) -> int:
        return len(self.indices)

    def entries(self) -> list:
        return list(zip(self.indices.tolist(), self.lengths.tolist()))

    @property
    def total_length(self) -> float:
        return float(self.lengths.sum())


def _angle_tables(geometry: ScanGeometry, dev):
    import torch
    cs = torch.tensor([math.cos(a) for a in geometry.angles], dtype=torch.float64, device=dev)
    sn = torch.tensor([math.sin(a) for a in geometry.angles], dtype=torch.float64, device=dev)
    return cs, sn


def siddon_csr(geometry: ScanGeometry, k0: int = 0, k1: int | None = None, dev=None):
    """Device CSR of the rays of views [k0, k1): (indptr i64, indices i32,
    values f64), rows k*N + c relative to k0."""
    import torch
    dev = dev or device()
    k1 = geometry.num_angles if k1 is None else k1
    n = geometry.num_detector_cols
    cs, sn = _angle_tables(geometry, dev)
    rays = (k1 - k0) * n
    counts = torch.empty(rays, dtype=torch.int64, device=dev)
    st = _lib.stream_handle(dev)
    _lib.call("xct_siddon_count", _lib.ptr(cs), _lib.ptr(sn), k0, k1, n, geometry.grid_n,
              float(geometry.voxel_size), _lib.ptr(counts), st)
    indptr = torch.zeros(rays + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=indptr[1:])
    nnz = int(indptr[-1].item())
    indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
    values = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)[:nnz]
    if nnz:
        _lib.call("xct_siddon_fill", _lib.ptr(cs), _lib.ptr(sn), k0, k1, n, geometry.grid_n,
                  float(geometry.voxel_size), _lib.ptr(indptr), _lib.ptr(indices),
                  _lib.ptr(values), st)
    return indptr, indices, values


def trace_ray(geometry: ScanGeometry, angle_index: int, detector_col: int) -> RaySegmentList:
    """Siddon trace of one ray (src/geometry.py:117-164), on the device."""
    if not 0 <= angle_index < geometry.num_angles:
        raise ValueError(f"angle_index {angle_index} out of range")
    if not 0 <= detector_col < geometry.num_detector_cols:
        raise ValueError(f"detector_col {detector_col} out of range")
    ip, idx, val = siddon_csr(geometry, angle_index, angle_index + 1)
    s, e = int(ip[detector_col]), int(ip[detector_col + 1])
    return RaySegmentList(idx[s:e].cpu().numpy().astype(np.int64), val[s:e].cpu().numpy())


class SystemMatrix:
    """Canonical CSR operator, device resident (src/geometry.py:167-195).

    ``indptr``/``indices``/``values`` are host numpy views created on first
    access (int64/int64/float64, as the reference returns); ``d_indptr``,
    ``d_indices``, ``d_values`` are the device arrays the builders use.
    """

    def __init__(self, num_rows, num_cols, num_angles, num_detector_cols,
                 d_indptr, d_indices, d_values):
        self.num_rows, self.num_cols = num_rows, num_cols
        self.num_angles, self.num_detector_cols = num_angles, num_detector_cols
        self.d_indptr, self.d_indices, self.d_values = d_indptr, d_indices, d_values
        self._nnz = int(d_indices.numel())
        self._host = None
        self._host32 = None

    def release_device(self) -> None:
        """Drop the device CSR (keeps host copies if already materialized)."""
        self.d_indptr = self.d_indices = self.d_values = None

    @classmethod
    def from_host(cls, num_rows, num_cols, indptr, indices, values, num_angles=None,
                  num_detector_cols=None):
        import torch
        dev = device()
        m = cls(num_rows, num_cols, num_angles or num_rows, num_detector_cols or 1,
                torch.as_tensor(np.asarray(indptr, np.int64), device=dev),
                torch.as_tensor(np.asarray(indices, np.int32), device=dev),
                torch.as_tensor(np.asarray(values, np.float64), device=dev))
        m._host = (np.asarray(indptr, np.int64), np.asarray(indices, np.int64),
                   np.asarray(values, np.float64))
        return m

    def _h32(self):
        """(indptr i64, indices i32, values f64) host copies, fetched once."""
        if getattr(self, "_host32", None) is None:
            if self._host is not None:
                ip, ix, v = self._host
                self._host32 = (ip, ix.astype(np.int32), v)
            else:
                self._host32 = (_lib.to_host(self.d_indptr), _lib.to_host(self.d_indices),
                                _lib.to_host(self.d_values))
        return self._host32

    def _h(self):
        if self._host is None:
            ip, ix, v = self._h32()
            self._host = (ip, ix.astype(np.int64), v)
        return self._host

    @property
    def indptr(self) -> np.ndarray:
        return self._h()[0]

    @property
    def indices(self) -> np.ndarray:
        return self._h()[1]

    @property
    def values(self) -> np.ndarray:
        return self._h()[2]

    @property
    def nnz(self) -> int:
        return self._nnz

    def host_csr32(self):
        """(indptr i64, indices i32, values f64) host arrays for the builders."""
        return self._h32()

    def row(self, r: int) -> RaySegmentList:
        s, e = self.indptr[r], self.indptr[r + 1]
        return RaySegmentList(self.indices[s:e], self.values[s:e])

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.num_rows, self.num_cols))
        row_of = np.repeat(np.arange(self.num_rows), np.diff(self.indptr))
        dense[row_of, self.indices] = self.values
        return dense


_matrix_cache: dict = {}
_build_counts: dict = {}


def build_system_matrix(geometry: ScanGeometry) -> SystemMatrix:
    """Memoized device build of the system matrix (src/geometry.py:202-232)."""
    cached = _matrix_cache.get(geometry)
    if cached is not None:
        return cached
    ip, idx, val = siddon_csr(geometry)
    m = SystemMatrix(geometry.num_rays, geometry.num_voxels, geometry.num_angles,
                     geometry.num_detector_cols, ip, idx, val)
    _matrix_cache[geometry] = m
    _build_counts[geometry] = _build_counts.get(geometry, 0) + 1
    return m


def clear_matrix_cache() -> None:
    _matrix_cache.clear()
    _build_counts.clear()


def build_count(geometry: ScanGeometry) -> int:
    return _build_counts.get(geometry, 0)


@dataclass
class Volume:
    """(slices, rows, cols) payload tagged tomogram/sinogram
    (src/geometry.py:245-273)."""

    data: np.ndarray
    role: str

    def __post_init__(self):
        if self.role not in ("tomogram", "sinogram"):
            raise ValueError(f"unknown volume role {self.role!r}")
        if self.data.ndim != 3:
            raise ValueError("volume payload must be 3D (slices, rows, cols)")

    @property
    def num_slices(self) -> int:
        return self.data.shape[0]

    @property
    def slice_shape(self):
        return self.data.shape[1], self.data.shape[2]

    def slices_as_columns(self) -> np.ndarray:
        return self.data.reshape(self.num_slices, -1).T

    @property
    def dtype_tag(self) -> str:
        return {np.float64: "double", np.float32: "single", np.float16: "half"}[
            self.data.dtype.type]


# head-phantom ellipses rescaled into [0, 1]: (value, a, b, x0, z0, degrees)
_ELLIPSES = ((1.00, 0.69, 0.92, 0.0, 0.0, 0.0), (-0.80, 0.6624, 0.8740, 0.0, -0.0184, 0.0),
             (-0.20, 0.1100, 0.3100, 0.22, 0.0, -18.0), (-0.20, 0.1600, 0.4100, -0.22, 0.0, 18.0),
             (0.10, 0.2100, 0.2500, 0.0, 0.35, 0.0), (0.10, 0.0460, 0.0460, 0.0, 0.1, 0.0),
             (0.10, 0.0460, 0.0460, 0.0, -0.1, 0.0), (0.10, 0.0460, 0.0230, -0.08, -0.605, 0.0),
             (0.10, 0.0230, 0.0230, 0.0, -0.606, 0.0), (0.10, 0.0230, 0.0460, 0.06, -0.605, 0.0))


def _grid(n):
    c = (n - 1) / 2.0
    iz, ix = np.mgrid[0:n, 0:n]
    return c, iz, ix


def _disk(n):
    c, iz, ix = _grid(n)
    return (ix - c) ** 2 + (iz - c) ** 2 <= (n / 2.0) ** 2


def generate_phantom(kind: str, grid_n: int, num_slices: int, seed: int = 0) -> Volume:
    """Synthetic tomogram in [0, 1], zero outside the inscribed circle
    (src/geometry.py:276-344).  Input synthesis, host side."""
    if kind not in PHANTOM_KINDS:
        raise ValueError(f"unknown phantom kind {kind!r}; expected one of {PHANTOM_KINDS}")
    if grid_n < 1 or num_slices < 1:
        raise ValueError("grid_n and num_slices must be >= 1")
    mask = _disk(grid_n)
    c, iz, ix = _grid(grid_n)
    if kind == "uniform-disk":
        base = np.ones((grid_n, grid_n)) * mask
        data = np.repeat(base[None], num_slices, axis=0)
    elif kind == "shepp-logan-like":
        x, z = (ix - c) / (grid_n / 2.0), (iz - c) / (grid_n / 2.0)
        img = np.zeros((grid_n, grid_n))
        for val, a, b, x0, z0, deg in _ELLIPSES:
            phi = math.radians(deg)
            xr = (x - x0) * math.cos(phi) + (z - z0) * math.sin(phi)
            zr = (z - z0) * math.cos(phi) - (x - x0) * math.sin(phi)
            img[(xr / a) ** 2 + (zr / b) ** 2 <= 1.0] += val
        data = np.repeat((np.clip(img, 0.0, 1.0) * mask)[None], num_slices, axis=0)
    else:
        rng = np.random.default_rng(seed)
        slices = []
        for _ in range(num_slices):
            img = np.zeros((grid_n, grid_n))
            for _ in range(6):
                bx, bz = rng.uniform(-0.6, 0.6, size=2) * (grid_n / 2.0)
                sigma = rng.uniform(0.08, 0.25) * grid_n
                amp = rng.uniform(0.3, 1.0)
                img += amp * np.exp(-(((ix - c - bx) ** 2 + (iz - c - bz) ** 2) / (2 * sigma**2)))
            peak = img.max()
            if peak > 0:
                img /= peak
            slices.append(img * mask)
        data = np.stack(slices)
    return Volume(np.ascontiguousarray(data), role="tomogram")


def simulate_measurements(matrix: SystemMatrix, tomogram: Volume, noise_sigma: float = 0.0,
                          seed: int = 0) -> Volume:
    """y = A x per slice in float64 on the device, plus optional Gaussian
    noise sigma*max(y) from numpy's seeded PCG64 (src/geometry.py:347-367)."""
    if tomogram.role != "tomogram":
        raise ValueError("expected a tomogram volume")
    rows, cols = tomogram.slice_shape
    if rows * cols != matrix.num_cols:
        raise ValueError(
            f"slice size {rows * cols} does not match matrix columns {matrix.num_cols}")
    from .engine import csr_spmm_f64
    y = csr_spmm_f64(matrix, tomogram.slices_as_columns().astype(np.float64))
    if noise_sigma > 0.0:
        rng = np.random.default_rng(seed)
        y = y + rng.normal(0.0, noise_sigma * y.max(), size=y.shape)
    data = y.T.reshape(tomogram.num_slices, matrix.num_angles, matrix.num_detector_cols)
    return Volume(np.ascontiguousarray(data), role="sinogram")


def project_f64(geometry: ScanGeometry, x: np.ndarray, chunk_nnz: float = 4e8) -> np.ndarray:
    """y = A x in float64 without holding A: Siddon regenerated per chunk of
    views on the device, each chunk multiplied by K-CSR-f64 (used for large
    geometries where build_system_matrix would not fit)."""
    import torch
    dev = device()
    X = np.ascontiguousarray(x.reshape(x.shape[0], -1), np.float64)
    d_x = torch.from_numpy(X).to(dev)
    n = geometry.grid_n
    per = max(1, int(chunk_nnz // (1.2 * n * n)))
    out = np.empty((geometry.num_rays, X.shape[1]))
    st = _lib.stream_handle(dev)
    for k0 in range(0, geometry.num_angles, per):
        k1 = min(geometry.num_angles, k0 + per)
        ip, ix, v = siddon_csr(geometry, k0, k1, dev)
        rows = (k1 - k0) * n
        y = torch.empty((rows, X.shape[1]), dtype=torch.float64, device=dev)
        _lib.call("xct_csr_spmm_f64", ip.data_ptr(), ix.data_ptr() if ix.numel() else None,
                  v.data_ptr() if v.numel() else None, rows, d_x.data_ptr(), X.shape[1],
                  y.data_ptr(), st)
        out[k0 * n:k1 * n] = y.cpu().numpy()
    return out.reshape(geometry.num_rays) if x.ndim == 1 else out


def project_matrix_free_f32(geometry: ScanGeometry, data, adjoint: bool = False):
    """Matrix-free single-precision projection of one chunk of 16 slices on
    the device (K11 ``xct_siddon_project_f32``): the Siddon rays are traced
    on the fly, no operator is stored.  ``data``: CUDA float32 tensor
    (num_voxels, 16) for the projection, (num_rays, 16) for the back
    projection (adjoint=True).  An independent FP32 implementation of the
    operator, used to check the staged path where an FP32 staged operator
    would not fit (bench.py, 2048^2 x 2048 views)."""
    import torch
    if not (isinstance(data, torch.Tensor) and data.is_cuda and data.dtype == torch.float32):
        raise ValueError("project_matrix_free_f32 expects a CUDA float32 tensor")
    n_in = geometry.num_rays if adjoint else geometry.num_voxels
    n_out = geometry.num_voxels if adjoint else geometry.num_rays
    if tuple(data.shape) != (n_in, 16):
        raise ValueError(f"expected shape ({n_in}, 16), got {tuple(data.shape)}")
    dev = data.device
    key = (geometry, str(dev))
    tabs = _MF_TABLES.get(key)
    if tabs is None:
        tabs = _MF_TABLES[key] = _angle_tables(geometry, dev)
    cs, sn = tabs
    x = data.contiguous()
    out = torch.zeros((n_out, 16), dtype=torch.float32, device=dev)
    _lib.call("xct_siddon_project_f32", _lib.ptr(cs), _lib.ptr(sn), 0, geometry.num_angles,
              geometry.num_detector_cols, geometry.grid_n, float(geometry.voxel_size),
              int(bool(adjoint)), x.data_ptr(), out.data_ptr(), _lib.stream_handle(dev))
    return out


_MF_TABLES: dict = {}
