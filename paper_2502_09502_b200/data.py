"""Synthetic inputs for the engine's parity cases and benchmark configs.

Host-side harness code (input generation is not on the hot path).  The
generator reproduces the reference's synthetic protocol bit for bit so that
the GPU engine and the CPU oracle see identical inputs:

* ``true_support``  — /root/reference/pkg/src/l0cert/data.py:63-73
* ``ar1_rows``      — data.py:76-85 (AR(1) rows, Toeplitz correlation sigma^|i-j|),
  evaluated in place on the Gaussian draw: every element is still
  ``sigma*x_{j-1} + c*w_j`` with the same two roundings, so the bits agree
  with the reference while peak memory halves.
* ``synthetic``     — data.py:88-115 (``generate_synthetic``: beta*, SNR noise
  with the reference's "variance" reading, labels)
* ``standardize``   — data.py:224-242

``make_config(name)`` builds the five BASELINE configs.

Instance ingest (same names, arguments, file formats
and errors as the reference's ``l0cert.data``): ``SyntheticParams`` /
``generate_synthetic`` (data.py:36-115), ``load_dataset`` (delimited and
libsvm-style sparse text, data.py:122-202), ``StandardizeTransform`` /
``standardize`` (data.py:205-242; a CUDA tensor is standardized on the
device), ``write_instance`` / ``read_instance`` (the ``l0cert-instance``
text format, data.py:248-317).
"""

from __future__ import annotations

import dataclasses
import math
import re
from typing import List, Optional, Tuple

import numpy as np

from .errors import DataFormatError, InvalidInputError

__all__ = [
    "true_support", "ar1_rows", "synthetic", "standardize", "ConfigData",
    "make_config", "CONFIGS", "random_nodes", "SyntheticParams", "generate_synthetic",
    "load_dataset", "StandardizeTransform", "write_instance", "read_instance",
    "DEFAULT_M", "DEFAULT_LAMBDA2",
]

DEFAULT_M = 2.0          # data.py:30-31 (benchmark defaults of generated instances)
DEFAULT_LAMBDA2 = 1.0


def true_support(p: int, k_true: int) -> np.ndarray:
    """0-based equally spaced support — data.py:63-73."""
    if p % k_true == 0:
        pos = np.arange(1, k_true + 1) * (p // k_true)
    else:
        pos = np.unique(np.round(np.arange(1, k_true + 1) * p / k_true).astype(np.int64))
        pos = np.clip(pos, 1, p)
    return pos - 1


def ar1_rows(n: int, p: int, sigma: float, rng: np.random.Generator,
             dtype=np.float64) -> np.ndarray:
    """Rows ~ N(0, Toeplitz(sigma^|i-j|)) by the AR(1) recursion — data.py:76-85.

    The recursion runs in place on the Gaussian draw (float64 arithmetic);
    ``dtype=np.float32`` rounds the finished matrix once, as the fp32 configs
    specify ("X cast to fp32").
    """
    X = rng.standard_normal((n, p))
    if sigma != 0.0:
        c = np.sqrt(1.0 - sigma * sigma)
        # the recursion is elementwise per row, so blocks of rows run it on a
        # transposed (column-contiguous) copy: the same roundings, without the
        # strided column walk over the whole matrix
        R = 512
        tmp = np.empty(R)
        for r0 in range(0, n, R):
            blk = np.ascontiguousarray(X[r0:r0 + R].T)     # p x rows
            t = tmp[:blk.shape[1]]
            for j in range(1, p):
                col = blk[j]
                np.multiply(col, c, out=t)                  # c * w_j
                np.multiply(blk[j - 1], sigma, out=col)     # sigma * x_{j-1}
                np.add(col, t, out=col)
            X[r0:r0 + R] = blk.T
    if dtype != np.float64:
        X = X.astype(dtype)
    return X


def synthetic(n: int, p: int, k_true: int, sigma: float = 0.5, snr: float = 5.0,
              seed: int = 0, task: str = "regression", snr_scale: str = "variance"):
    """(X, y, beta_true) of ``generate_synthetic`` — data.py:88-115."""
    rng = np.random.default_rng(seed)
    X = ar1_rows(n, p, sigma, rng)
    beta_true = np.zeros(p)
    beta_true[true_support(p, k_true)] = 1.0
    signal = X @ beta_true
    scale = np.linalg.norm(signal) / snr
    noise_std = np.sqrt(scale) if snr_scale == "variance" else scale
    eps = rng.normal(0.0, noise_std, n) if noise_std > 0 else np.zeros(n)
    if task == "regression":
        y = signal + eps
    else:
        prob = np.clip(signal + eps, 0.0, 1.0)
        y = np.where(rng.random(n) < prob, 1.0, -1.0)
    return X, y, beta_true


@dataclasses.dataclass
class StandardizeTransform:
    """What ``standardize`` did (data.py:205-221): kept / dropped columns, the
    kept columns' means and centred norms."""
    kept: np.ndarray
    dropped: np.ndarray
    means: np.ndarray
    norms: np.ndarray

    def map_coefficients(self, beta_std) -> Tuple[np.ndarray, float]:
        """Coefficients of the standardized problem on the original scale (zero
        at dropped columns) and the intercept shift of the centring."""
        b = np.asarray(beta_std, dtype=np.float64) / self.norms
        out = np.zeros(self.kept.size + self.dropped.size)
        out[self.kept] = b
        return out, float(-(self.means @ b))


def standardize(X):
    """Centre every column, scale it to unit Euclidean norm, drop the constant
    ones (data.py:224-242).  Returns (X_std, StandardizeTransform); a CUDA
    tensor is processed on its device and returned as one."""
    try:
        import torch
        on_gpu = isinstance(X, torch.Tensor) and X.device.type == "cuda"
    except ImportError:  # pragma: no cover
        on_gpu = False
    if on_gpu:
        # hand-written kernels (csrc/standardize.cu), bit-identical to the
        # numpy branch below: sequential column sums over rows, as numpy
        # reduces a C-contiguous matrix over axis 0
        import ctypes
        from . import _device, native
        if X.ndim != 2 or X.shape[0] < 2:
            raise InvalidInputError("standardize needs a 2-d matrix with n >= 2")
        Xd = X.to(torch.float64).contiguous()
        n, p = Xd.shape
        lib = native.load()
        stats = torch.empty((3, p), dtype=torch.float64, device=Xd.device)
        st = _device.stream_handle()
        native.check(lib.l0_standardize_stats(Xd.data_ptr(), n, p, p, stats[0].data_ptr(),
                                              stats[1].data_ptr(), stats[2].data_ptr(), st))
        means, norms, scale = stats.cpu().numpy()
        keep = norms > 1e-12 * np.maximum(1.0, scale)
        if not keep.any():
            raise InvalidInputError("all columns are constant")
        kept = np.nonzero(keep)[0]
        kd = torch.from_numpy(kept.astype(np.int64)).to(Xd.device)
        out = torch.empty((n, kept.size), dtype=torch.float64, device=Xd.device)
        native.check(lib.l0_standardize_apply(Xd.data_ptr(), n, p, kd.data_ptr(), kept.size,
                                              stats[0].data_ptr(), stats[1].data_ptr(), out.data_ptr(), st))
        return out, StandardizeTransform(kept=kept, dropped=np.nonzero(~keep)[0],
                                         means=means[kept], norms=norms[kept])
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] < 2:
        raise InvalidInputError("standardize needs a 2-d matrix with n >= 2")
    means = X.mean(axis=0)
    centered = X - means
    norms = np.linalg.norm(centered, axis=0)
    scale = np.abs(X).max(axis=0)
    keep = norms > 1e-12 * np.maximum(1.0, scale)
    if not keep.any():
        raise InvalidInputError("all columns are constant")
    kept = np.nonzero(keep)[0]
    return centered[:, kept] / norms[kept], StandardizeTransform(
        kept=kept, dropped=np.nonzero(~keep)[0], means=means[kept], norms=norms[kept])


@dataclasses.dataclass
class SyntheticParams:
    """data.py:36-60 (validated on construction)."""
    n: int
    p: int
    k_true: int
    sigma: float = 0.5
    snr: float = 5.0
    task: str = "regression"
    seed: int = 0
    snr_scale: str = "variance"

    def __post_init__(self):
        if self.n < 1 or self.p < 1:
            raise InvalidInputError("n and p must be positive")
        if not 1 <= self.k_true <= self.p:
            raise InvalidInputError("k_true must satisfy 1 <= k_true <= p")
        if not 0.0 <= self.sigma < 1.0:
            raise InvalidInputError("sigma must lie in [0, 1)")
        if not self.snr > 0:
            raise InvalidInputError("snr must be positive")
        if self.task not in ("regression", "classification"):
            raise InvalidInputError("task must be 'regression' or 'classification'")
        if self.snr_scale not in ("variance", "std"):
            raise InvalidInputError("snr_scale must be 'variance' or 'std'")


def generate_synthetic(params: SyntheticParams):
    """The seeded instance of data.py:88-115 (cardinality k_true, M and
    lambda2 at the benchmark defaults, ground truth attached)."""
    from .model import LossKind, ProblemInstance
    X, y, bt = synthetic(params.n, params.p, params.k_true, params.sigma, params.snr,
                         params.seed, params.task, params.snr_scale)
    loss = LossKind.SQUARED_ERROR if params.task == "regression" else LossKind.LOGISTIC
    return ProblemInstance(X=X, y=y, loss=loss, k=params.k_true, M=DEFAULT_M,
                           lambda2=DEFAULT_LAMBDA2, beta_true=bt)


_FIELD_SPLIT = re.compile(r"[,\s]+")


def _data_lines(path):
    """(line number, stripped text) of the non-blank, non-comment lines."""
    with open(path) as fh:
        for no, raw in enumerate(fh, start=1):
            text = raw.strip()
            if text and not text.startswith("#"):
                yield no, text


def load_dataset(path, fmt: str = "delimited", label_column: str = "last",
                 n_features: Optional[int] = None):
    """(X, y) from a text file (data.py:122-202).  ``delimited``: one sample per
    line, comma or whitespace separated, the label first or last;
    ``sparse``: ``label idx:value ...`` with 1-based feature indices."""
    if fmt not in ("delimited", "sparse"):
        raise InvalidInputError(f"unknown dataset format {fmt!r}")
    if label_column not in ("last", "first"):
        raise InvalidInputError("label_column must be 'last' or 'first'")
    if fmt == "delimited":
        X, y, width = [], [], None
        for no, text in _data_lines(path):
            parts = [f for f in _FIELD_SPLIT.split(text) if f]
            if width is None:
                if len(parts) < 2:
                    raise DataFormatError(f"line {no}: need at least one feature and a label", line=no)
                width = len(parts)
            elif len(parts) != width:
                raise DataFormatError(f"line {no}: expected {width} fields, found {len(parts)}", line=no)
            try:
                vals = [float(f) for f in parts]
            except ValueError as exc:
                raise DataFormatError(f"line {no}: {exc}", line=no) from None
            if label_column == "last":
                X.append(vals[:-1]); y.append(vals[-1])
            else:
                X.append(vals[1:]); y.append(vals[0])
        if not X:
            raise DataFormatError("file contains no data rows")
        return np.asarray(X, dtype=np.float64), np.asarray(y, dtype=np.float64)
    samples, top = [], 0
    for no, text in _data_lines(path):
        parts = text.split()
        try:
            lab = float(parts[0])
            feats = []
            for tok in parts[1:]:
                j_s, v_s = tok.split(":", 1)
                j = int(j_s)
                if j < 1:
                    raise ValueError(f"feature index {j} is not 1-based")
                feats.append((j, float(v_s)))
        except (ValueError, IndexError) as exc:
            raise DataFormatError(f"line {no}: {exc}", line=no) from None
        top = max([top] + [j for j, _ in feats])
        samples.append((lab, feats))
    if not samples:
        raise DataFormatError("file contains no data rows")
    width = n_features if n_features is not None else top
    if top > width:
        raise DataFormatError(f"feature index {top} exceeds declared width {width}")
    X = np.zeros((len(samples), width))
    y = np.empty(len(samples))
    for i, (lab, feats) in enumerate(samples):
        y[i] = lab
        for j, v in feats:
            X[i, j - 1] = v
    return X, y


def write_instance(path, instance) -> None:
    """The ``l0cert-instance`` text format (data.py:248-266): a key/value
    header, ``data``, then one sample per line with the label last; the
    ground-truth support is written 1-based.  Floats round-trip (repr)."""
    X = np.asarray(instance.X, dtype=np.float64) if not hasattr(instance.X, "cpu") else \
        instance.X.detach().cpu().numpy().astype(np.float64)
    y = np.asarray(instance.y, dtype=np.float64)
    lines = ["format l0cert-instance 1", f"n {X.shape[0]}", f"p {X.shape[1]}",
             f"loss {instance.loss.value}", f"k {instance.k}", f"M {float(instance.M)!r}",
             f"lambda2 {float(instance.lambda2)!r}"]
    if instance.beta_true is not None:
        sup = np.flatnonzero(np.asarray(instance.beta_true)) + 1
        lines.append("support_true " + ",".join(str(int(j)) for j in sup))
    lines.append("data")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
        for i in range(X.shape[0]):
            fh.write(" ".join(repr(float(v)) for v in X[i]) + f" {float(y[i])!r}\n")


def _num(tok: str) -> float:
    # the reference's writer emits numpy-2 reprs for numpy scalars
    # ("np.float64(-1.0)", data.py:266); accept them so its files load here
    if tok.startswith("np.float64(") and tok.endswith(")"):
        tok = tok[len("np.float64("):-1]
    return float(tok)


def read_instance(path):
    """Inverse of ``write_instance`` (data.py:269-317); also reads files the
    reference wrote under numpy 2 (labels as ``np.float64(...)`` reprs)."""
    from .model import LossKind, ProblemInstance
    head, rows, body = {}, [], False
    for no, text in _data_lines(path):
        if not body:
            if text == "data":
                body = True
                continue
            kv = text.split(None, 1)
            if len(kv) != 2:
                raise DataFormatError(f"line {no}: malformed header line", line=no)
            head[kv[0]] = kv[1].strip()
            continue
        try:
            rows.append([_num(f) for f in text.split()])
        except ValueError as exc:
            raise DataFormatError(f"line {no}: {exc}", line=no) from None
    for key in ("n", "p", "loss", "k", "M", "lambda2"):
        if key not in head:
            raise DataFormatError(f"missing header field {key!r}")
    n, p = int(head["n"]), int(head["p"])
    names = {kind.value: kind for kind in LossKind}
    if head["loss"] not in names:
        raise DataFormatError(f"unknown loss {head['loss']!r}")
    if len(rows) != n:
        raise DataFormatError(f"header declares n={n} but found {len(rows)} data rows")
    if any(len(r) != p + 1 for r in rows):
        raise DataFormatError(f"every data row needs p + 1 = {p + 1} fields")
    A = np.asarray(rows, dtype=np.float64).reshape(n, p + 1)
    bt = None
    if "support_true" in head and head["support_true"]:
        bt = np.zeros(p)
        bt[[int(j) - 1 for j in head["support_true"].split(",")]] = 1.0
    return ProblemInstance(X=A[:, :p], y=A[:, p], loss=names[head["loss"]], k=int(head["k"]),
                           M=float(head["M"]), lambda2=float(head["lambda2"]), beta_true=bt)


@dataclasses.dataclass
class ConfigData:
    name: str
    X: np.ndarray            # host matrix (float64, or float32 for the fp32 configs)
    y: np.ndarray            # float64 labels
    loss: str                # "squared_error" | "logistic"
    k: int
    M: float
    lambda2: float
    iterations: Optional[int]    # fixed iteration count (None: run to the gap)
    rel_gap: Optional[float]     # relative gap target (C2)
    dtype: str                   # "fp64" | "fp32"
    beta_true: Optional[np.ndarray] = None
    nodes: Optional[list] = None  # [(fixed_zero, fixed_one)] for C4
    note: str = ""

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def p(self) -> int:
        return self.X.shape[1]


def random_nodes(p: int, count: int, seed: int = 1, max_zero: int = 8, max_one: int = 4):
    """C4's seeded node sets: per node nz ~ U{0..8},
    no ~ U{0..4}, disjoint indices drawn without replacement."""
    rng = np.random.default_rng(seed)
    nodes = []
    for _ in range(count):
        nz = int(rng.integers(0, max_zero + 1))
        no = int(rng.integers(0, max_one + 1))
        idx = rng.choice(p, nz + no, replace=False)
        nodes.append((tuple(sorted(int(i) for i in idx[:nz])),
                      tuple(sorted(int(i) for i in idx[nz:]))))
    return nodes


def _c1(scale: float = 1.0, literal: bool = False) -> ConfigData:
    n, p = int(2000 * scale), int(1000 * scale)
    if literal:
        # the reference pipeline verbatim: y from the raw X, then standardize X
        X, y, bt = synthetic(n, p, 10, sigma=0.5, snr=5.0, seed=0)
        Xs, _ = standardize(X)
        note = "literal reference pipeline (degenerate: gap hits 0 at t=10)"
    else:
        rng = np.random.default_rng(0)
        Xs, _ = standardize(ar1_rows(n, p, 0.5, rng))
        bt = np.zeros(p)
        bt[true_support(p, 10)] = 1.0
        sig = Xs @ bt
        eps = rng.normal(0.0, math.sqrt(np.linalg.norm(sig) / 5.0), n)
        y = sig + eps
        note = "y drawn from the standardised X (well-posed)"
    return ConfigData("C1" + ("-literal" if literal else ""), np.ascontiguousarray(Xs), y,
                      "squared_error", 10, 2.0, 1.0, 1000, None, "fp64", bt, note=note)


def _c2(scale: float = 1.0) -> ConfigData:
    n = p = int(16000 * scale)
    X, y, bt = synthetic(n, p, 20, sigma=0.7, snr=5.0, seed=0)
    return ConfigData("C2", X, y, "squared_error", 20, 2.0, 0.1, None, 1e-6, "fp64", bt)


def _c3(scale: float = 1.0) -> ConfigData:
    n, p = int(50000 * scale), int(20000 * scale)
    rng = np.random.default_rng(0)
    X = ar1_rows(n, p, 0.5, rng, dtype=np.float32)
    bt = np.zeros(p)
    bt[true_support(p, 15)] = 1.0
    eta = X.astype(np.float64) @ bt
    prob = 1.0 / (1.0 + np.exp(-eta))
    y = np.where(rng.random(n) < prob, 1.0, -1.0)
    return ConfigData("C3", X, y, "logistic", 15, 3.0, 0.01, 2000, None, "fp32", bt,
                      note="labels ~ Bernoulli(sigmoid(x.beta*)) (builder recipe)")


def _c4(scale: float = 1.0, nodes: int = 512) -> ConfigData:
    n, p = int(20000 * scale), int(5000 * scale)
    X, y, bt = synthetic(n, p, 10, sigma=0.5, snr=5.0, seed=0)
    return ConfigData("C4", X.astype(np.float32), y, "squared_error", 10, 2.0, 0.5, 500,
                      None, "fp32", bt, nodes=random_nodes(p, nodes, seed=1))


def _c5(scale: float = 1.0, block_rows: int = 100_000) -> ConfigData:
    n, p = int(1_000_000 * scale), int(10_000 * min(1.0, scale * 10))
    X = np.empty((n, p), dtype=np.float32)
    for b, r0 in enumerate(range(0, n, block_rows)):
        r1 = min(n, r0 + block_rows)
        X[r0:r1] = ar1_rows(r1 - r0, p, 0.5, np.random.default_rng([0, b]), dtype=np.float32)
    bt = np.zeros(p)
    bt[true_support(p, 25)] = 1.0
    sig = X.astype(np.float64) @ bt if n * p <= 2e8 else _rowblock_matvec(X, bt)
    eps = np.random.default_rng([0, 1 << 20]).normal(0.0, math.sqrt(np.linalg.norm(sig) / 5.0), n)
    return ConfigData("C5", X, sig + eps, "squared_error", 25, 2.0, 0.1, 1000, None, "fp32", bt)


def _rowblock_matvec(X, v, block=50_000):
    out = np.empty(X.shape[0])
    for r0 in range(0, X.shape[0], block):
        out[r0:r0 + block] = X[r0:r0 + block].astype(np.float64) @ v
    return out


CONFIGS = {"C1": _c1, "C1-literal": lambda scale=1.0: _c1(scale, literal=True),
           "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5}


def make_config(name: str, scale: float = 1.0, **kw) -> ConfigData:
    """Build config ``name`` (C1, C1-literal, C2, C3, C4, C5) at ``scale``
    (scale < 1 shrinks n and p proportionally for parity tests)."""
    return CONFIGS[name](scale=scale, **kw) if kw else CONFIGS[name](scale=scale)


# ---------------------------------------------------------------------------
# C5 on the device (bench): AR(1) rows generated in HBM, sharded by rows
# ---------------------------------------------------------------------------
C5_N, C5_P, C5_BLOCK = 1_000_000, 10_000, 100_000


def ar1_block_device(b: int, rows: int, p: int, sigma: float, device, seed: int = 0):
    """Rows of generator block ``b`` of an AR(1) design (Toeplitz sigma^|i-j|
    correlation, N(0, 1) marginals; the recursion of data.py:76-85) drawn on
    the device from torch's Philox generator seeded (seed, b), fp32, as a
    (p, rows) column-major block.  Blocks are independent of how rows are
    later sharded, so every world size sees the same matrix."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed((seed << 32) + b)
    W = torch.randn((p, rows), generator=g, device=device, dtype=torch.float32)
    if sigma != 0.0:
        c = math.sqrt(1.0 - sigma * sigma)
        for j in range(1, p):
            W[j].mul_(c).add_(W[j - 1], alpha=sigma)
    return W


def c5_shard_device(r0: int, r1: int, device, n: int = C5_N, p: int = C5_P, k_true: int = 25,
                    sigma: float = 0.5, snr: float = 5.0, block: int = C5_BLOCK, allreduce=None):
    """Rows [r0, r1) of C5 (n x p fp32, Toeplitz 0.5, k=25 evenly spaced ones,
    SNR 5) built on ``device``: X (rows x p, row-major fp32) and y (fp64).
    The noise scale needs ||X beta*|| over all n rows: ``allreduce`` sums a
    1-element CUDA tensor over the ranks (None on one rank)."""
    import torch
    rows = r1 - r0
    X = torch.empty((rows, p), dtype=torch.float32, device=device)
    for b in range(r0 // block, (r1 - 1) // block + 1):
        b0, b1 = b * block, min(n, (b + 1) * block)
        lo, hi = max(r0, b0), min(r1, b1)
        W = ar1_block_device(b, b1 - b0, p, sigma, device)
        X[lo - r0:hi - r0].copy_(W[:, lo - b0:hi - b0].T)
        del W
    support = torch.from_numpy(true_support(p, k_true)).to(device)
    sig = X.index_select(1, support).to(torch.float64).sum(1)        # X beta* (beta* = 1 on S)
    sq = (sig * sig).sum().reshape(1)
    if allreduce is not None:
        allreduce(sq)
    std = math.sqrt(math.sqrt(float(sq.item())) / snr)                # data.py:97-99 "variance"
    eps = torch.empty(rows, dtype=torch.float64, device=device)
    for b in range(r0 // block, (r1 - 1) // block + 1):
        b0, b1 = b * block, min(n, (b + 1) * block)
        lo, hi = max(r0, b0), min(r1, b1)
        g = torch.Generator(device=device)
        g.manual_seed((1 << 40) + b)
        e = torch.randn(b1 - b0, generator=g, device=device, dtype=torch.float64) * std
        eps[lo - r0:hi - r0] = e[lo - b0:hi - b0]
    return X, sig + eps
