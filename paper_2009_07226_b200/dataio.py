"""Dataset container (XCT1), PGM slice export, CSV reports and run manifests
-- the data formats on either side of the hot path.

Same file formats, names and error behaviour as the reference's
``xct.dataio`` (src/dataio.py:30-163), so datasets written by either
package read back bit-identically in the other (pinned by
``tests/golden/xct1_*`` fixtures written with the reference).

XCT1 layout (little endian):
    b"XCT1" | u8 dtype (0 f64, 1 f32, 2 f16) | u8 role (0 tomogram,
    1 sinogram) | u8 ndim | ndim x u32 dims | row-major payload
Tomograms are (slice, z, x), sinograms (slice, angle, detector); slices
are contiguous, so a slice range is one contiguous byte range.
"""

from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from .geometry import Volume

__all__ = ["DatasetFormatError", "write_volume", "read_volume", "read_slices", "write_pgm",
           "write_csv", "RunManifest", "sha256_of"]

MAGIC = b"XCT1"
_HEAD = struct.Struct("<4sBBB")
_CODE_OF = {np.dtype(np.float64): 0, np.dtype(np.float32): 1, np.dtype(np.float16): 2}
_DTYPE_OF = {c: d.newbyteorder("<") for d, c in _CODE_OF.items()}
_ROLES = ("tomogram", "sinogram")


class DatasetFormatError(ValueError):
    """The file is not a well-formed dataset container."""


def write_volume(path, volume: Volume) -> None:
    """Header + payload in one write (src/dataio.py:36-52)."""
    data = volume.data
    code = _CODE_OF.get(data.dtype.newbyteorder("="))
    if code is None:
        raise DatasetFormatError(f"unsupported dtype {data.dtype}")
    head = _HEAD.pack(MAGIC, code, _ROLES.index(volume.role), data.ndim)
    dims = struct.pack(f"<{data.ndim}I", *data.shape)
    payload = np.ascontiguousarray(data, dtype=_DTYPE_OF[code])
    with open(path, "wb") as fh:
        fh.write(head + dims)
        fh.write(memoryview(payload).cast("B"))


def _parse_header(path: Path, raw: bytes):
    if len(raw) < _HEAD.size or raw[:4] != MAGIC:
        raise DatasetFormatError(f"{path}: bad magic (expected XCT1)")
    _, code, role, ndim = _HEAD.unpack_from(raw)
    if code not in _DTYPE_OF:
        raise DatasetFormatError(f"{path}: unknown dtype code {code}")
    if role >= len(_ROLES):
        raise DatasetFormatError(f"{path}: unknown role code {role}")
    end = _HEAD.size + 4 * ndim
    if len(raw) < end:
        raise DatasetFormatError(f"{path}: truncated header")
    dims = struct.unpack_from(f"<{ndim}I", raw, _HEAD.size)
    return _DTYPE_OF[code], _ROLES[role], dims, end


def read_volume(path) -> Volume:
    """Parse and validate a container (src/dataio.py:55-82): missing file ->
    FileNotFoundError naming it; bad magic / codes / sizes ->
    DatasetFormatError."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"dataset file not found: {path}")
    raw = path.read_bytes()
    dtype, role, dims, end = _parse_header(path, raw)
    want = int(np.prod(dims, dtype=np.int64)) * dtype.itemsize
    if len(raw) - end != want:
        raise DatasetFormatError(f"{path}: payload is {len(raw) - end} bytes, expected {want}")
    data = np.frombuffer(raw, dtype=dtype, offset=end).reshape(dims)
    return Volume(data=data.astype(dtype.newbyteorder("=")), role=role)


def read_slices(path, lo: int, hi: int) -> Volume:
    """Slices [lo, hi) of a 3D container without reading the rest of the
    payload (the layout keeps slices contiguous; a slice-batch rank reads
    only its own group, src/cli.py:158-200)."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"dataset file not found: {path}")
    with open(path, "rb") as fh:
        head = fh.read(_HEAD.size + 4 * 8)
        dtype, role, dims, end = _parse_header(path, head)
        if len(dims) != 3 or not 0 <= lo <= hi <= dims[0]:
            raise ValueError(f"{path}: slice range [{lo}, {hi}) outside {dims}")
        per = dims[1] * dims[2] * dtype.itemsize
        fh.seek(end + lo * per)
        buf = fh.read((hi - lo) * per)
    if len(buf) != (hi - lo) * per:
        raise DatasetFormatError(f"{path}: truncated payload")
    data = np.frombuffer(buf, dtype=dtype).reshape(hi - lo, dims[1], dims[2])
    return Volume(data=data.astype(dtype.newbyteorder("=")), role=role)


def write_pgm(path, image: np.ndarray) -> None:
    """16-bit binary PGM of one slice, min-max windowed to 0..65535
    (constant images are all black), src/dataio.py:85-99."""
    if image.ndim != 2:
        raise ValueError("PGM export needs a 2D slice")
    img = np.asarray(image, dtype=np.float64)
    lo, hi = float(img.min()), float(img.max())
    # same operation order as the reference (difference / range, then x 65535)
    level = np.round((img - lo) / (hi - lo) * 65535.0) if hi > lo else np.zeros(img.shape)
    head = b"P5\n%d %d\n65535\n" % (img.shape[1], img.shape[0])
    Path(path).write_bytes(head + level.astype(">u2").tobytes())


def write_csv(path, header: list[str], rows: list) -> None:
    """ASCII CSV; floats as %.9e (src/dataio.py:102-112)."""
    def cell(v):
        return f"{v:.9e}" if isinstance(v, float) else str(v)
    text = "\n".join([",".join(header)] + [",".join(cell(v) for v in r) for r in rows])
    Path(path).write_text(text + "\n", encoding="ascii")


def sha256_of(path) -> str:
    return hashlib.sha256(Path(path).read_bytes()).hexdigest()


@dataclass
class RunManifest:
    """Everything needed to re-run a command bit-identically
    (src/dataio.py:121-163); saved as sorted, indented JSON."""

    command: str
    arguments: dict = field(default_factory=dict)
    seeds: dict = field(default_factory=dict)
    phase_seconds: dict = field(default_factory=dict)
    volume_report: dict = field(default_factory=dict)
    counters: dict = field(default_factory=dict)
    outputs: dict = field(default_factory=dict)
    residual_csv: str | None = None

    def add_output(self, path) -> None:
        self.outputs[str(path)] = sha256_of(path)

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(asdict(self), indent=2, sort_keys=True) + "\n",
                              encoding="ascii")

    @staticmethod
    def load(path) -> "RunManifest":
        d = json.loads(Path(path).read_text(encoding="ascii"))
        keys = RunManifest.__dataclass_fields__
        return RunManifest(**{k: v for k, v in d.items() if k in keys})
