"""Host-side problem synthesis and dataset files for the CLI.

Behavioural mirror of the reference's ``ladlasso.datagen`` / ``ladlasso.rng``
(datagen.py:28-140, rng.py:25-72): the same GenSpec fields and validation,
the same PCG32 stream (XSH-RR output, stream selector 54, Box-Muller normals
served cos-then-sin with the spare kept across phases, rejection-sampled
bounded integers) and the same draw order -- design row-major, informative
coefficients U[1,10], m noise normals (even when sigma is 0), outlier rows
until distinct -- so `generate(spec)` is bit-identical to the reference's on
the same host.  tests/test_cli.py pins it against the reference-generated
golden inputs (kat.npz stall case, acceptance.npz grid).

The dataset CSV format is the reference's: header ``x1,...,xd,y``, one point
per row, shortest round-trip float repr; plus a ``.meta.json`` sidecar.

The BASELINE.json config generators (configs 0-4) run on the device instead
(configgen.py); this module exists for the reference-facing CLI.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from .errors import InvalidInputError
from .solver import Coefficients, Dataset

__all__ = ["Pcg32", "GenSpec", "generate", "generate_batched", "write_dataset_csv", "read_dataset_csv", "metadata_path",
           "write_metadata", "read_metadata"]

_M64 = 0xFFFFFFFFFFFFFFFF
_M32 = 0xFFFFFFFF
_LCG_MUL = 6364136223846793005
_INV_2_32 = 1.0 / 4294967296.0  # exact power of two: u * 2^-32 == u / 2^32
_TAU = 2.0 * math.pi


class Pcg32:
    """PCG32 with the generator's sampling conventions (rng.py:25-72)."""

    __slots__ = ("_state", "_inc", "_spare")

    def __init__(self, seed: int, stream: int = 54):
        self._inc = (2 * stream + 1) & _M64
        self._state = 0
        self._step()
        self._state = (self._state + (seed & _M64)) & _M64
        self._step()
        self._spare = None

    def _step(self) -> int:
        """Advance the LCG; return the XSH-RR output of the previous state."""
        s = self._state
        self._state = (s * _LCG_MUL + self._inc) & _M64
        word = ((s ^ (s >> 18)) >> 27) & _M32
        rot = s >> 59
        if rot == 0:
            return word
        return ((word >> rot) | (word << (32 - rot))) & _M32

    def uniform(self) -> float:
        return self._step() * _INV_2_32

    def uniform_in(self, a: float, b: float) -> float:
        return a + (b - a) * self.uniform()

    def below(self, bound: int) -> int:
        if bound <= 0:
            raise ValueError("bound must be positive")
        reject_under = (1 << 32) % bound
        r = self._step()
        while r < reject_under:
            r = self._step()
        return r % bound

    def normal(self) -> float:
        spare = self._spare
        if spare is not None:
            self._spare = None
            return spare
        u_open = (self._step() + 1) * _INV_2_32  # (0, 1]
        u_half = self._step() * _INV_2_32  # [0, 1)
        rho = math.sqrt(-2.0 * math.log(u_open))
        theta = _TAU * u_half
        self._spare = rho * math.sin(theta)
        return rho * math.cos(theta)

    def normals(self, count: int) -> list[float]:
        draw = self.normal
        return [draw() for _ in range(count)]


def _require(ok: bool, message: str) -> None:
    if not ok:
        raise InvalidInputError(message)


@dataclass(frozen=True)
class GenSpec:
    """Generation recipe (datagen.py:28-62); `n_informative` None means all d axes."""

    m: int
    d: int
    n_informative: int | None = None
    true_coefficients: tuple[float, ...] | None = None
    noise_sigma: float = 1.0
    outlier_fraction: float = 0.0
    outlier_scale: float = 10.0
    seed: int = 0

    def __post_init__(self):
        _require(self.m >= 1 and self.d >= 1, "need m >= 1 and d >= 1")
        informative = self.d if self.n_informative is None else self.n_informative
        _require(1 <= informative <= self.d, f"n_informative must be in [1, {self.d}], got {informative}")
        if self.true_coefficients is not None:
            given = tuple(map(float, self.true_coefficients))
            _require(len(given) == self.d, "true_coefficients must have length d")
            object.__setattr__(self, "true_coefficients", given)
        _require(self.noise_sigma >= 0, "noise_sigma must be >= 0")
        _require(0 <= self.outlier_fraction < 1, "outlier_fraction must be in [0, 1)")
        _require(self.outlier_scale >= 1, "outlier_scale must be >= 1")
        object.__setattr__(self, "n_informative", informative)

    @property
    def n_outliers(self) -> int:
        return math.floor(self.outlier_fraction * self.m)


def generate(g: GenSpec) -> tuple[Dataset, Coefficients]:
    """(dataset, true coefficients) for `g`; a pure function of the spec (datagen.py:65-80)."""
    stream = Pcg32(g.seed)
    design = np.array(stream.normals(g.m * g.d)).reshape(g.m, g.d)
    if g.true_coefficients is None:
        truth = np.zeros(g.d)
        for j in range(g.n_informative):
            truth[j] = stream.uniform_in(1.0, 10.0)
    else:
        truth = np.array(g.true_coefficients)
    noise = np.array(stream.normals(g.m)) * g.noise_sigma
    outlier_rows: set[int] = set()
    want = g.n_outliers
    while len(outlier_rows) < want:
        outlier_rows.add(stream.below(g.m))
    # each chosen row is scaled exactly once, so the set's iteration order is immaterial
    rows = np.fromiter(outlier_rows, dtype=np.int64, count=len(outlier_rows))
    noise[rows] *= g.outlier_scale
    response = design @ truth + noise
    return Dataset(design, response), Coefficients(truth)


def generate_batched(specs, device="cuda"):
    """``generate`` for many GenSpecs at once ON THE DEVICE (lad_genspec_generate_f64, one
    thread per problem): returns CUDA tensors X (B, m, d), y (B, m), beta_true (B, d).  The
    specs may differ only in their seeds.  The transcendentals are double-double and rounded
    once, so the result equals ``generate`` wherever glibc's log/sin/cos are correctly rounded
    (all golden inputs; tests/test_gpu_genspec.py bounds any difference: each transcendental within 1 ulp of glibc's, each normal draw within 2 ulp)."""
    import torch

    from . import _lib
    from .solver import _check

    specs = list(specs)
    if not specs:
        raise InvalidInputError("need at least one GenSpec")
    g0 = specs[0]
    key = lambda g: (g.m, g.d, g.n_informative, g.true_coefficients, g.noise_sigma, g.outlier_fraction,
                     g.outlier_scale)
    if any(key(g) != key(g0) for g in specs[1:]):
        raise InvalidInputError("generate_batched: specs must differ only in their seeds")
    dev = torch.device(device)
    B, m, d = len(specs), g0.m, g0.d
    seeds = torch.from_numpy(np.array([g.seed & _M64 for g in specs], dtype=np.uint64).view(np.int64)).to(dev)
    X = torch.empty((B, m, d), dtype=torch.float64, device=dev)
    y = torch.empty((B, m), dtype=torch.float64, device=dev)
    bt = torch.empty((B, d), dtype=torch.float64, device=dev)
    truth = None
    if g0.true_coefficients is not None:
        truth = torch.tensor(g0.true_coefficients, dtype=torch.float64, device=dev)
    _check(_lib.load().lad_genspec_generate_f64(
        B, m, d, g0.n_informative, truth.data_ptr() if truth is not None else None, float(g0.noise_sigma),
        float(g0.outlier_fraction), float(g0.outlier_scale), seeds.data_ptr(), X.data_ptr(), y.data_ptr(),
        bt.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    return X, y, bt


def _csv_header(d: int) -> str:
    return ",".join([f"x{j}" for j in range(1, d + 1)] + ["y"])


def write_dataset_csv(data: Dataset, path) -> None:
    """Reference CSV layout (datagen.py:83-89): values written with repr() so they round-trip."""
    x, y = data.x, data.y
    body = [",".join(map(repr, map(float, x[i]))) + "," + repr(float(y[i])) for i in range(data.m)]
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join([_csv_header(data.d)] + body) + "\n")


def read_dataset_csv(path) -> Dataset:
    """Parse a dataset CSV with the reference's error messages (datagen.py:92-121)."""
    with open(path, "r", encoding="ascii") as fh:
        text = fh.read().split("\n")
    if text and text[-1] == "":
        text.pop()
    if not text:
        raise InvalidInputError(f"{path}: empty file")
    columns = text[0].split(",")
    width = len(columns)
    if width < 2 or text[0] != _csv_header(width - 1):
        raise InvalidInputError(f"{path}: header row 1 must be x1,...,xd,y, got {text[0]!r}")
    table = []
    for lineno, line in enumerate(text[1:], start=2):
        if not line:
            continue
        cells = line.split(",")
        if len(cells) != width:
            raise InvalidInputError(f"{path}: row {lineno} has {len(cells)} fields, header has {width}")
        values = []
        for col, cell in enumerate(cells):
            try:
                values.append(float(cell))
            except ValueError:
                raise InvalidInputError(
                    f"{path}: row {lineno}, column {columns[col]}: cannot parse {cell!r} as a number") from None
        table.append(values)
    if not table:
        raise InvalidInputError(f"{path}: no data rows")
    arr = np.array(table)
    return Dataset(arr[:, :-1], arr[:, -1])


def metadata_path(csv_path) -> str:
    return f"{csv_path}.meta.json"


def write_metadata(csv_path, g: GenSpec, true_beta: Coefficients) -> None:
    """Sidecar JSON: the GenSpec fields plus ``true_beta`` (datagen.py:128-135)."""
    record = dict(asdict(g), true_beta=[float(v) for v in true_beta.beta])
    with open(metadata_path(csv_path), "w", encoding="ascii") as fh:
        fh.write(json.dumps(record, indent=2, sort_keys=True) + "\n")


def read_metadata(csv_path) -> dict:
    with open(metadata_path(csv_path), "r", encoding="ascii") as fh:
        return json.load(fh)
