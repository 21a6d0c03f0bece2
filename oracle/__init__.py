"""oracle -- TEST INFRASTRUCTURE ONLY: the CPU parity checker.

Two checkers, both fp64 and both following the reference's CPU path
(/root/reference/proj, arxiv 2308.00497):

* ``Oracle``  -- ctypes binding of ``oracle/libfftgen_oracle.so``, the plain-C
  restatement in ``oracle/fftgen_oracle.c`` (pinned bit-exact against the
  reference's own outputs by tests/test_oracle.py).
* ``Ref``     -- ctypes binding of ``oracle/_ref/libfftgen_ref.so``: the
  UNMODIFIED reference library compiled in place by ``oracle/Makefile`` plus
  the thin forwarding shim ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` arm may import this package.  The product package
(``paper_2308_00497_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libfftgen_oracle.so")
AOT_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libref_aot.so")
REF_SO = os.path.join(HERE, "_ref", "libfftgen_ref.so")

ALG = {"cooley-tukey": 0, "ct": 0, "stockham": 1}
LAYOUT = {"interleaved": 0, "split": 1}
KIND_NAMES = {0: "FusedMKIV", 1: "FusedIKMV", 2: "FusedPKIV", 3: "TwiddleMul", 4: "Permute", 5: "DenseApply"}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def build(quiet: bool = True) -> None:
    """Build both checkers (the reference part only if its tree is present)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


def _alg(a) -> int:
    return ALG[a] if isinstance(a, str) else int(a)


def _lay(layout) -> int:
    return LAYOUT[layout] if isinstance(layout, str) else int(layout)


class OrcOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("p0", C.c_int64), ("p1", C.c_int64), ("p2", C.c_int64),
                ("tw_total", C.c_int64), ("tw_block", C.c_int64), ("tw_repeat", C.c_int64)]


def as_complex(inter: np.ndarray) -> np.ndarray:
    return inter[..., 0::2] + 1j * inter[..., 1::2]


def as_interleaved(z: np.ndarray) -> np.ndarray:
    out = np.empty(z.shape[:-1] + (2 * z.shape[-1],), dtype=np.float64)
    out[..., 0::2] = z.real
    out[..., 1::2] = z.imag
    return out


class Oracle:
    """Plain-C restatement (oracle/fftgen_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_seeded_input.argtypes = [C.c_int64, C.c_uint64, _dp]
        L.orc_unit_root.argtypes = [C.c_int64, C.c_int64, _dp]
        L.orc_stockham_radices.argtypes = [C.c_int64, C.c_int64, _i64p, C.c_int]
        L.orc_fuse.argtypes = [C.c_int64, C.c_int, C.c_int64, C.POINTER(OrcOp), C.c_int]
        L.orc_op_index_map.argtypes = [C.POINTER(OrcOp), C.c_int64, _i64p]
        L.orc_op_twiddle_exps.argtypes = [C.POINTER(OrcOp), C.c_int64, _i64p]
        for f in (L.orc_forward_batch, L.orc_inverse_batch):
            f.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int64, _dp, _dp, C.c_int]
        L.orc_dft_oracle.argtypes = [C.c_int64, _dp, _dp]
        L.orc_dft_bins.argtypes = [C.c_int64, _dp, C.c_int64, _i64p, C.c_int, _dp]
        L.orc_error_metric.argtypes = [C.c_int64, _dp, _dp]
        L.orc_error_metric.restype = C.c_double
        L.orc_mflops.argtypes = [C.c_int64, C.c_double]
        L.orc_mflops.restype = C.c_double
        L.orc_last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc < 0:
            raise RuntimeError(f"oracle error {rc}: {self.lib.orc_last_error().decode()}")
        return rc

    def seeded_input(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(2 * n, dtype=np.float64)
        self.lib.orc_seeded_input(n, seed, _ptr(out))
        return out

    def unit_root(self, n: int, t: int) -> complex:
        out = np.empty(2, dtype=np.float64)
        self.lib.orc_unit_root(n, t, _ptr(out))
        return complex(out[0], out[1])

    def stockham_radices(self, n: int, radix: int) -> list[int]:
        buf = np.zeros(64, dtype=np.int64)
        cnt = self._check(self.lib.orc_stockham_radices(n, radix, _ptr(buf, _i64p), 64))
        return [int(v) for v in buf[:cnt]]

    def fuse(self, n: int, alg, radix: int) -> list[OrcOp]:
        ops = (OrcOp * 4096)()
        cnt = self._check(self.lib.orc_fuse(n, _alg(alg), radix, ops, 4096))
        return [ops[i] for i in range(cnt)]

    def pipeline_text(self, n: int, alg, radix: int) -> str:
        lines = []
        for op in self.fuse(n, alg, radix):
            if op.kind == 0:
                lines.append(f"FusedMKIV(m={op.p0}, copies={op.p1})")
            elif op.kind == 1:
                lines.append(f"FusedIKMV(n={op.p0}, copies={op.p1})")
            elif op.kind == 2:
                lines.append(f"FusedPKIV(m={op.p0}, total={op.p1}, k={op.p2})")
            elif op.kind == 3:
                lines.append(f"TwiddleMul(len={n})")
            else:
                lines.append(f"Permute(m={op.p0}, total={op.p1})")
        return "".join(l + "\n" for l in lines)

    def op_index_map(self, op: OrcOp, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        self._check(self.lib.orc_op_index_map(C.byref(op), n, _ptr(out, _i64p)))
        return out

    def op_twiddle_exps(self, op: OrcOp, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        self._check(self.lib.orc_op_twiddle_exps(C.byref(op), n, _ptr(out, _i64p)))
        return out

    def forward(self, x: np.ndarray, alg="stockham", radix: int = 4, threads: int = 1,
                inverse: bool = False) -> np.ndarray:
        """x: (batch, 2n) or (2n,) interleaved float64 -> same shape."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        flat = x.reshape(-1, x.shape[-1])
        n = flat.shape[1] // 2
        out = np.empty_like(flat)
        fn = self.lib.orc_inverse_batch if inverse else self.lib.orc_forward_batch
        self._check(fn(n, _alg(alg), radix, flat.shape[0], _ptr(flat), _ptr(out), threads))
        return out.reshape(x.shape)

    def dft_oracle(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self.lib.orc_dft_oracle(x.shape[0] // 2, _ptr(x), _ptr(out))
        return out

    def dft_bins(self, x: np.ndarray, bins, inverse: bool = False) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.ascontiguousarray(np.asarray(bins, dtype=np.int64))
        out = np.empty(2 * b.shape[0], dtype=np.float64)
        self.lib.orc_dft_bins(x.shape[0] // 2, _ptr(x), b.shape[0], _ptr(b, _i64p),
                              1 if inverse else -1, _ptr(out))
        return out

    def error_metric(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return self.lib.orc_error_metric(a.shape[0] // 2, _ptr(a), _ptr(b))

    def mflops(self, n: int, seconds: float) -> float:
        return self.lib.orc_mflops(n, seconds)


class Ref:
    """The unmodified reference library (oracle/_ref/libfftgen_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: build it with `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_seeded_input.argtypes = [C.c_int64, C.c_uint64, _dp]
        L.ref_unit_root.argtypes = [C.c_int64, C.c_int64, _dp]
        L.ref_dft_oracle.argtypes = [C.c_int64, _dp, _dp]
        L.ref_forward_batch.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_int64, _dp, _dp, C.c_int]
        L.ref_compile.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int]
        L.ref_formula_text.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_char_p, C.c_int64]
        L.ref_pipeline_text.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_char_p, C.c_int64]
        L.ref_num_ops.argtypes = [C.c_int64, C.c_int, C.c_int64]
        L.ref_op_desc.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int, _i64p]
        L.ref_op_index_map.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int, _i64p]
        L.ref_op_twiddle.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_int64, _i64p, _dp]
        L.ref_emit_c.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_char_p, C.c_char_p,
                                 C.c_int64, _i64p]
        L.ref_mflops.argtypes = [C.c_int64, C.c_double]
        L.ref_mflops.restype = C.c_double
        L.ref_error_metric.argtypes = [C.c_int64, _dp, _dp]
        L.ref_error_metric.restype = C.c_double

    ERRORS = {1: "PlanError", 2: "DimensionError", 3: "ExecError", 4: "Error", 5: "std::exception"}

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"{self.ERRORS.get(rc, rc)}: {self.lib.ref_last_error().decode()}")

    def seeded_input(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(2 * n, dtype=np.float64)
        self._check(self.lib.ref_seeded_input(n, seed, _ptr(out)))
        return out

    def unit_root(self, n: int, t: int) -> complex:
        out = np.empty(2, dtype=np.float64)
        self.lib.ref_unit_root(n, t, _ptr(out))
        return complex(out[0], out[1])

    def dft_oracle(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self.lib.ref_dft_oracle(x.shape[0] // 2, _ptr(x), _ptr(out)))
        return out

    def forward(self, x: np.ndarray, alg="cooley-tukey", radix: int = 2, layout="interleaved",
                threads: int = 1) -> np.ndarray:
        """compile_pipeline + interpret; x is (batch, 2n) or (2n,) in the given
        ComplexBuffer layout (split = [re n | im n] per transform)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        flat = x.reshape(-1, x.shape[-1])
        n = flat.shape[1] // 2
        out = np.empty_like(flat)
        self._check(self.lib.ref_forward_batch(n, _alg(alg), radix, _lay(layout), flat.shape[0],
                                               _ptr(flat), _ptr(out), threads))
        return out.reshape(x.shape)

    def compile(self, n: int, alg="cooley-tukey", radix: int = 2, layout="interleaved") -> None:
        self._check(self.lib.ref_compile(n, _alg(alg), radix, _lay(layout)))

    def formula_text(self, n: int, alg, radix: int) -> str:
        buf = C.create_string_buffer(1 << 20)
        self._check(self.lib.ref_formula_text(n, _alg(alg), radix, buf, len(buf)))
        return buf.value.decode()

    def pipeline_text(self, n: int, alg, radix: int) -> str:
        buf = C.create_string_buffer(1 << 22)
        self._check(self.lib.ref_pipeline_text(n, _alg(alg), radix, buf, len(buf)))
        return buf.value.decode()

    def num_ops(self, n: int, alg, radix: int) -> int:
        return self.lib.ref_num_ops(n, _alg(alg), radix)

    def op_desc(self, n: int, alg, radix: int, idx: int) -> tuple:
        d = np.zeros(4, dtype=np.int64)
        self._check(self.lib.ref_op_desc(n, _alg(alg), radix, idx, _ptr(d, _i64p)))
        return tuple(int(v) for v in d)

    def op_index_map(self, n: int, alg, radix: int, idx: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        self._check(self.lib.ref_op_index_map(n, _alg(alg), radix, idx, _ptr(out, _i64p)))
        return out

    def op_twiddle(self, n: int, alg, radix: int, idx: int, s: int):
        exps = np.empty(n, dtype=np.int64)
        coeffs = np.empty(2 * n, dtype=np.float64)
        self._check(self.lib.ref_op_twiddle(n, _alg(alg), radix, idx, s, _ptr(exps, _i64p),
                                            _ptr(coeffs)))
        return exps, coeffs

    def emit_c(self, n: int, alg, radix: int, layout="interleaved", fn: str = "fft") -> str:
        ln = np.zeros(1, dtype=np.int64)
        self._check(self.lib.ref_emit_c(n, _alg(alg), radix, _lay(layout), fn.encode(), None, 0,
                                        _ptr(ln, _i64p)))
        buf = C.create_string_buffer(int(ln[0]) + 1)
        self._check(self.lib.ref_emit_c(n, _alg(alg), radix, _lay(layout), fn.encode(), buf,
                                        len(buf), _ptr(ln, _i64p)))
        return buf.value.decode()

    def mflops(self, n: int, seconds: float) -> float:
        return self.lib.ref_mflops(n, seconds)


class AotRef:
    """The reference's ahead-of-time C path (emit_c output for N=4096,
    Stockham radix 4, split layout) with a batch-parallel driver
    (oracle/_ref/libref_aot.so, built by oracle/build_aot.py).  Baseline
    infrastructure only: bench.py's cpu_baseline leg and tests."""

    N, ALG, RADIX, LAYOUT = 4096, "stockham", 4, "split"

    def __init__(self, path: str = AOT_SO):
        self.lib = C.CDLL(path)
        self.lib.ref_aot_batch.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int]
        self.lib.ref_aot_batch.restype = C.c_int

    def forward(self, x: np.ndarray, threads: int = 1) -> np.ndarray:
        """x: (batch, 2N) float64 in the split ComplexBuffer layout [re N | im N]."""
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 2 * self.N)
        y = np.empty_like(x)
        rc = self.lib.ref_aot_batch(_ptr(x), _ptr(y), x.shape[0], self.N, threads)
        if rc != 0:
            raise RuntimeError("ref_aot_batch failed")
        return y


def relayout_to_split(inter: np.ndarray) -> np.ndarray:
    """interleaved (.., 2n) -> reference split ComplexBuffer (.., [re n | im n])."""
    return np.concatenate([inter[..., 0::2], inter[..., 1::2]], axis=-1)


def split_to_interleaved(split: np.ndarray) -> np.ndarray:
    n = split.shape[-1] // 2
    out = np.empty_like(split)
    out[..., 0::2] = split[..., :n]
    out[..., 1::2] = split[..., n:]
    return out


def rel_l2(got: np.ndarray, want: np.ndarray) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm((got - want).ravel()) / np.linalg.norm(want.ravel()))
