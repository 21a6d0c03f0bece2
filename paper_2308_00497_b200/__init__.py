"""paper_2308_00497_b200 -- B200-native batched 1-D complex FFT (FFTc hot path).

Python binding (ctypes) of the C ABI in ``include/fftgen_b200.h``; it mirrors
the reference's plan -> execute API (``/root/reference/proj/include/fftgen``):

    reference (C++)                         here
    PipelineConfig  driver.hpp:26-35        PipelineConfig (+ batch, device)
    compile_pipeline driver.hpp:44-45       compile_pipeline() -> Plan
    interpret        exec.hpp:26-27         Plan.execute (device tensors),
                                            Plan.execute_host (host fp32),
                                            interpret() (fp64 ComplexBuffer storage)
    print_pipeline   rewrite.hpp:91-92      Plan.pipeline_text()
    Error classes    error.hpp:16-71        FftgenError / PlanError / ...

The compute path is the sm_100a library ``lib/libfftgen_b200.so``.  There is
no CPU fallback: if the library is missing, importing this package raises.
PyTorch is only used (optionally) to pass device pointers and streams.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libfftgen_b200.so")
CSRC = os.path.join(HERE, "csrc")

FORWARD = -1
INVERSE = 1
LAYOUTS = {"interleaved": 0, "split": 1}
ALGORITHMS = {"cooley-tukey": 0, "ct": 0, "stockham": 1}
OP_NAMES = {0: "FusedMKIV", 1: "FusedIKMV", 2: "FusedPKIV", 3: "TwiddleMul", 4: "Permute"}

# Symbols the C ABI header declares (tests check the library exports each).
ABI_SYMBOLS = (
    "fftgen_config_init", "fftgen_plan_create", "fftgen_plan_destroy", "fftgen_execute",
    "fftgen_execute_host", "fftgen_interpret_f64", "fftgen_error_string", "fftgen_last_error",
    "fftgen_abi_version", "fftgen_plan_radices", "fftgen_plan_num_ops", "fftgen_plan_op",
    "fftgen_plan_op_map", "fftgen_plan_pipeline_text", "fftgen_plan_num_passes", "fftgen_plan_pass",
    "fftgen_plan_describe", "fftgen_plan_launches", "fftgen_plan_scratch_bytes",
    "fftgen_twiddle_multiply",
)


class FftgenError(RuntimeError):
    """Base class, like fftgen::Error (error.hpp:16-19)."""


class PlanError(FftgenError):
    """Invalid planner request (error.hpp:38-41)."""


class DimensionError(FftgenError):
    """Sizes do not line up (error.hpp:32-35)."""


class FuseError(FftgenError):
    """Kernel above the fusion cap (error.hpp:44-47)."""


class ExecError(FftgenError):
    """Runtime failure while executing (error.hpp:56-59)."""


_STATUS = {1: PlanError, 2: DimensionError, 3: ExecError, 4: FuseError, 5: DimensionError,
           6: ExecError, 7: ExecError}


class _Config(C.Structure):
    _fields_ = [("n", C.c_int64), ("algorithm", C.c_int32), ("radix", C.c_int32),
                ("layout", C.c_int32), ("device", C.c_int32), ("batch", C.c_int64)]


def build(jobs: int = 8, quiet: bool = True) -> str:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-C", CSRC, f"-j{jobs}"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i64, i64p = C.c_void_p, C.c_int64, C.POINTER(C.c_int64)
    L.fftgen_config_init.argtypes = [C.POINTER(_Config)]
    L.fftgen_config_init.restype = None
    L.fftgen_plan_create.argtypes = [C.POINTER(vp), C.POINTER(_Config)]
    L.fftgen_plan_destroy.argtypes = [vp]
    L.fftgen_execute.argtypes = [vp, C.c_int, vp, vp, vp, vp, i64, vp]
    L.fftgen_execute_host.argtypes = [vp, C.c_int, vp, vp, vp, vp, i64]
    L.fftgen_interpret_f64.argtypes = [vp, C.c_int, vp, vp]
    L.fftgen_error_string.argtypes = [C.c_int]
    L.fftgen_error_string.restype = C.c_char_p
    L.fftgen_last_error.restype = C.c_char_p
    L.fftgen_plan_radices.argtypes = [vp, i64p, C.c_int]
    L.fftgen_plan_num_ops.argtypes = [vp]
    L.fftgen_plan_op.argtypes = [vp, C.c_int, i64p]
    L.fftgen_plan_op_map.argtypes = [vp, C.c_int, i64p, i64p]
    L.fftgen_plan_pipeline_text.argtypes = [vp, C.c_char_p, C.c_size_t]
    L.fftgen_plan_num_passes.argtypes = [vp]
    L.fftgen_plan_pass.argtypes = [vp, C.c_int, i64p]
    L.fftgen_plan_describe.argtypes = [vp, C.c_char_p, C.c_size_t]
    L.fftgen_plan_launches.argtypes = [vp]
    L.fftgen_plan_scratch_bytes.argtypes = [vp]
    L.fftgen_plan_scratch_bytes.restype = C.c_size_t
    L.fftgen_twiddle_multiply.argtypes = [C.c_int, vp, i64, i64, i64, i64, i64, i64, vp]
    return L


lib = _load()


def _check(status: int) -> None:
    if status != 0:
        cls = _STATUS.get(status, FftgenError)
        raise cls(f"{lib.fftgen_error_string(status).decode()}: {lib.fftgen_last_error().decode()}")


@dataclass
class PipelineConfig:
    """Mirror of fftgen::PipelineConfig (driver.hpp:26-35) plus batch/device."""
    n: int = 0
    algorithm: str = "cooley-tukey"
    radix: int = 2
    layout: str = "interleaved"
    batch: int = 1
    device: int = 0


def _ptr(x) -> int:
    """Device/host address of a torch tensor or numpy array (None -> 0)."""
    if x is None:
        return 0
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, np.ndarray):
        return int(x.ctypes.data)
    return int(x)


class Plan:
    """A compiled plan (CompiledPipeline analogue); owns device twiddle tables."""

    def __init__(self, cfg: PipelineConfig):
        self.config = cfg
        c = _Config()
        lib.fftgen_config_init(C.byref(c))
        c.n = int(cfg.n)
        c.algorithm = ALGORITHMS[cfg.algorithm] if isinstance(cfg.algorithm, str) else int(cfg.algorithm)
        c.radix = int(cfg.radix)
        c.layout = LAYOUTS[cfg.layout] if isinstance(cfg.layout, str) else int(cfg.layout)
        c.batch = int(cfg.batch)
        c.device = int(cfg.device)
        h = C.c_void_p()
        _check(lib.fftgen_plan_create(C.byref(h), C.byref(c)))
        self._h = h
        self.n = c.n
        self.batch = c.batch
        self.split = c.layout == 1

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.fftgen_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- execution ------------------------------------------------------
    def execute(self, in0, out0, in1=None, out1=None, direction: int = FORWARD,
                dist: Optional[int] = None, stream=None) -> None:
        """Device execute.  Interleaved: float32 tensors (batch, dist, 2) or
        complex64; split: re/im float32 tensors (batch, dist).  `stream` is a
        torch.cuda.Stream, a raw cudaStream_t int, or None (current stream)."""
        if dist is None:
            dist = self.n
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(self.config.device).cuda_stream
            except Exception:
                stream = 0
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        _check(lib.fftgen_execute(self._h, direction, _ptr(in0), _ptr(in1), _ptr(out0), _ptr(out1),
                                  int(dist), int(stream)))

    def execute_host(self, in0: np.ndarray, out0: np.ndarray, in1=None, out1=None,
                     direction: int = FORWARD, dist: Optional[int] = None) -> None:
        """Host fp32 buffers (numpy or pinned CPU tensors); pipelined H2D/compute/D2H."""
        for a in (in0, out0, in1, out1):
            if isinstance(a, np.ndarray) and (a.dtype != np.float32 or not a.flags.c_contiguous):
                raise DimensionError("host buffers must be C-contiguous float32")
        _check(lib.fftgen_execute_host(self._h, direction, _ptr(in0), _ptr(in1), _ptr(out0), _ptr(out1),
                                       int(dist if dist is not None else self.n)))

    def interpret(self, x: np.ndarray, direction: int = FORWARD) -> np.ndarray:
        """fp64 ComplexBuffer storage in/out: (batch, 2n) doubles in the plan layout."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != 2 * self.n * self.batch:
            raise DimensionError(f"input holds {x.size} doubles, plan needs {2 * self.n * self.batch}")
        out = np.empty_like(x)
        _check(lib.fftgen_interpret_f64(self._h, direction, _ptr(x), _ptr(out)))
        return out

    # ---- introspection --------------------------------------------------
    def radices(self) -> list[int]:
        buf = (C.c_int64 * 64)()
        cnt = lib.fftgen_plan_radices(self._h, buf, 64)
        return [int(buf[i]) for i in range(cnt)]

    def ops(self) -> list[tuple]:
        out = []
        d = (C.c_int64 * 4)()
        for i in range(lib.fftgen_plan_num_ops(self._h)):
            _check(lib.fftgen_plan_op(self._h, i, d))
            out.append(tuple(int(v) for v in d))
        return out

    def op_map(self, idx: int):
        m = np.empty(self.n, dtype=np.int64)
        s = C.c_int64(0)
        _check(lib.fftgen_plan_op_map(self._h, idx, m.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(s)))
        return m, int(s.value)

    def pipeline_text(self) -> str:
        buf = C.create_string_buffer(1 << 22)
        _check(lib.fftgen_plan_pipeline_text(self._h, buf, len(buf)))
        return buf.value.decode()

    def passes(self) -> list[tuple]:
        out = []
        d = (C.c_int64 * 4)()
        for i in range(lib.fftgen_plan_num_passes(self._h)):
            _check(lib.fftgen_plan_pass(self._h, i, d))
            out.append(tuple(int(v) for v in d))
        return out

    def describe(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        _check(lib.fftgen_plan_describe(self._h, buf, len(buf)))
        return buf.value.decode()

    def launches(self) -> int:
        return int(lib.fftgen_plan_launches(self._h))

    def scratch_bytes(self) -> int:
        return int(lib.fftgen_plan_scratch_bytes(self._h))


def compile_pipeline(cfg: PipelineConfig) -> Plan:
    """compile_pipeline (driver.cpp:11-34) analogue: validate, plan, upload twiddles."""
    return Plan(cfg)


def interpret(plan: Plan, x: np.ndarray, direction: int = FORWARD) -> np.ndarray:
    """interpret(final_ir, ComplexBuffer) analogue on fp64 reference storage."""
    return plan.interpret(x, direction)


def twiddle_multiply(block, row_offset: int, col_offset: int, n: int, direction: int = FORWARD,
                     stream=None) -> None:
    """In place on a CUDA complex64 (rows, cols) block (or float32 (rows, cols, 2)):
    block[r, c] *= w_n^{(row_offset + r)(col_offset + c)} -- the four-step
    twiddle diagonal D^N (formula.hpp:44-49) on one rank's block."""
    rows, cols = block.shape[0], block.shape[1]
    ld = block.stride(0) if block.dtype.is_complex else block.stride(0) // 2
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(block.device).cuda_stream
    _check(lib.fftgen_twiddle_multiply(direction, _ptr(block), rows, cols, ld, row_offset, col_offset, n,
                                       int(stream)))


def flops(n: int, batch: int = 1) -> float:
    """5 N log2 N per transform (verify.cpp:48-51)."""
    return 5.0 * n * np.log2(n) * batch if n > 1 else 0.0
