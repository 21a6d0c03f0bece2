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
    "fftgen_twiddle_multiply", "fftgen_dist_plan_create", "fftgen_dist_plan_destroy", "fftgen_dist_butterfly",
    "fftgen_dist_local", "fftgen_dist_unpack", "fftgen_dist_execute", "fftgen_dist_chunk_elems",
    "fftgen_dist_block_elems", "fftgen_dist_local_plan", "fftgen_seeded_input", "fftgen_program_text",
    "fftgen_plan_group_twiddles", "fftgen_dist_butterfly_peers", "fftgen_dist_unpack_peers",
    "fftgen_dist_execute_cyclic",
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


class LowerError(FftgenError):
    """A schedule option was rejected (error.hpp:50-53)."""


class BoundsError(FftgenError):
    """A buffer is shorter than the plan's access range (error.hpp:62-65)."""


class GpuMapError(FftgenError):
    """No launch geometry for the plan on this device (error.hpp:68-71)."""


_STATUS = {1: PlanError, 2: DimensionError, 3: ExecError, 4: FuseError, 5: DimensionError,
           6: ExecError, 7: ExecError, 8: LowerError, 9: BoundsError, 10: GpuMapError}

# fftgen_config.tuning bits (include/fftgen_b200.h)
TUNE_NO_TMA = 1
TUNE_NO_TMA_STORE = 2
TUNE_GROUP_TMA_ALL = 4
VEC_MODES = {"none": 0, "inner": 1, "outer": 2}


class _Config(C.Structure):
    _fields_ = [("n", C.c_int64), ("algorithm", C.c_int32), ("radix", C.c_int32),
                ("layout", C.c_int32), ("device", C.c_int32), ("batch", C.c_int64),
                ("vec", C.c_int32), ("vector_width", C.c_int32), ("interleaved_opt", C.c_int32),
                ("tile_kind", C.c_int32), ("tile_value", C.c_int64),
                ("tuning", C.c_uint32), ("cluster_size", C.c_int32), ("host_chunk_mb", C.c_int32),
                ("pass_radix", C.c_int32)]


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
    L.fftgen_abi_version.restype = C.c_int
    if L.fftgen_abi_version() != 3:
        raise ImportError(f"{LIB_PATH} has ABI {L.fftgen_abi_version()}, this binding needs 3: rebuild it")
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
    L.fftgen_dist_plan_create.argtypes = [C.POINTER(vp), i64, C.c_int, C.c_int, C.c_int]
    L.fftgen_dist_plan_destroy.argtypes = [vp]
    L.fftgen_dist_butterfly.argtypes = [vp, C.c_int, vp, vp, vp]
    L.fftgen_dist_local.argtypes = [vp, C.c_int, vp, vp, vp]
    L.fftgen_dist_unpack.argtypes = [vp, vp, vp, vp]
    L.fftgen_dist_execute.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp]
    L.fftgen_dist_execute_cyclic.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp]
    L.fftgen_dist_chunk_elems.argtypes = [vp]
    L.fftgen_dist_chunk_elems.restype = i64
    L.fftgen_dist_block_elems.argtypes = [vp]
    L.fftgen_dist_block_elems.restype = i64
    L.fftgen_dist_local_plan.argtypes = [vp]
    L.fftgen_dist_local_plan.restype = vp
    L.fftgen_seeded_input.argtypes = [C.c_int, i64, i64, C.c_uint64, vp, vp, i64, C.c_int, vp]
    L.fftgen_program_text.argtypes = [C.POINTER(_Config), C.c_int, C.c_char_p, C.c_size_t]
    L.fftgen_plan_group_twiddles.argtypes = [vp, C.c_int, C.c_int, vp, i64]
    L.fftgen_dist_butterfly_peers.argtypes = [vp, C.c_int, C.POINTER(vp), C.POINTER(vp), vp]
    L.fftgen_dist_unpack_peers.argtypes = [vp, C.POINTER(vp), vp, vp]
    L.fftgen_plan_group_twiddles.restype = i64
    return L


lib = _load()


def _check(status: int) -> None:
    if status != 0:
        cls = _STATUS.get(status, FftgenError)
        raise cls(f"{lib.fftgen_error_string(status).decode()}: {lib.fftgen_last_error().decode()}")


@dataclass
class PipelineConfig:
    """Mirror of fftgen::PipelineConfig (driver.hpp:26-35) plus batch/device.

    vec / vector_width / interleaved_opt / tile are the reference's CPU
    loop-IR schedule: validated like vectorize()/tile() (LowerError) and
    result-neutral.  tuning / cluster_size / host_chunk_mb select among the
    sm_100a kernels (0 = the measured defaults)."""
    n: int = 0
    algorithm: str = "cooley-tukey"
    radix: int = 2
    layout: str = "interleaved"
    batch: int = 1
    device: int = 0
    vec: str = "none"
    vector_width: int = 8
    interleaved_opt: bool = False
    tile: Optional[tuple] = None          # ("exact", size) or ("cache", bytes)
    tuning: int = 0
    cluster_size: int = 0
    host_chunk_mb: int = 0
    pass_radix: int = 0                   # radix hint for the register passes (0 = measured default)


def _ptr(x) -> int:
    """Device/host address of a torch tensor or numpy array (None -> 0)."""
    if x is None:
        return 0
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, np.ndarray):
        return int(x.ctypes.data)
    return int(x)


def _to_config(cfg: PipelineConfig) -> "_Config":
    """PipelineConfig -> the C ABI fftgen_config (driver.hpp:26-35 + B200 fields)."""
    c = _Config()
    lib.fftgen_config_init(C.byref(c))
    c.n = int(cfg.n)
    c.algorithm = ALGORITHMS[cfg.algorithm] if isinstance(cfg.algorithm, str) else int(cfg.algorithm)
    c.radix = int(cfg.radix)
    c.layout = LAYOUTS[cfg.layout] if isinstance(cfg.layout, str) else int(cfg.layout)
    c.batch = int(cfg.batch)
    c.device = int(cfg.device)
    c.vec = VEC_MODES[cfg.vec] if isinstance(cfg.vec, str) else int(cfg.vec)
    c.vector_width = int(cfg.vector_width)
    c.interleaved_opt = int(bool(cfg.interleaved_opt))
    if cfg.tile is not None:
        kind, value = cfg.tile
        c.tile_kind = {"exact": 1, "cache": 2}[kind]
        c.tile_value = int(value)
    c.tuning = int(cfg.tuning)
    c.cluster_size = int(cfg.cluster_size)
    c.host_chunk_mb = int(cfg.host_chunk_mb)
    c.pass_radix = int(cfg.pass_radix)
    return c


class Plan:
    """A compiled plan (CompiledPipeline analogue); owns device twiddle tables."""

    def __init__(self, cfg: PipelineConfig):
        self.config = cfg
        c = _to_config(cfg)
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
    def _check_buffers(self, bufs, dist: int, device: bool) -> None:
        """Device / dtype / layout / size of every buffer against the plan's
        access range: transform b, element e at b*dist + e (BoundsError when
        a buffer is shorter, like the reference's check_bounds)."""
        need = (self.batch - 1) * dist + self.n  # elements (complex for interleaved)
        for name, a in bufs:
            if a is None:
                continue
            if hasattr(a, "data_ptr"):  # torch tensor
                import torch
                if device:
                    if a.device.type != "cuda" or a.device.index != self.config.device:
                        raise ExecError(f"{name} is on {a.device}, plan is on cuda:{self.config.device}")
                elif a.device.type != "cpu":
                    raise ExecError(f"{name} must be a host (CPU) tensor, got {a.device}")
                if a.dtype == torch.complex64:
                    elems = a.numel()
                elif a.dtype == torch.float32:
                    elems = a.numel() // (1 if self.split else 2)
                else:
                    raise ExecError(f"{name} must be float32 or complex64, got {a.dtype}")
                if self.split and a.dtype != torch.float32:
                    raise ExecError(f"split layout takes float32 planes, {name} is {a.dtype}")
                per = 1 if (self.split or a.dtype == torch.complex64) else 2  # storage scalars per element
                if not a.is_contiguous():
                    # strided views are fine when they ARE the plan's addressing:
                    # one transform per leading index, dist elements apart
                    if a.dim() < 2 or not a[0].is_contiguous() or a.stride(0) != dist * per:
                        raise ExecError(f"{name} is a strided view that does not match dist={dist} "
                                        f"(stride {tuple(a.stride())})")
                avail = a.untyped_storage().nbytes() - a.storage_offset() * a.element_size()
                elems = avail // (a.element_size() * per)
            elif isinstance(a, np.ndarray):
                if device:
                    raise ExecError(f"{name} is a host array; use execute_host")
                if a.dtype == np.complex64:
                    elems = a.size
                elif a.dtype == np.float32:
                    elems = a.size // (1 if self.split else 2)
                else:
                    raise DimensionError(f"host buffers must be float32 or complex64, {name} is {a.dtype}")
                if not a.flags.c_contiguous:
                    raise DimensionError(f"{name} must be C-contiguous")
            else:
                continue  # raw address: the caller vouches for it
            if elems < need:
                raise BoundsError(f"{name} holds {elems} elements, the plan reads/writes {need} "
                                  f"(batch {self.batch}, dist {dist}, n {self.n})")

    def execute(self, in0, out0, in1=None, out1=None, direction: int = FORWARD,
                dist: Optional[int] = None, stream=None) -> None:
        """Device execute.  Interleaved: float32 tensors (batch, dist, 2) or
        complex64; split: re/im float32 tensors (batch, dist).  `stream` is a
        torch.cuda.Stream, a raw cudaStream_t int, or None (current stream)."""
        if dist is None:
            dist = self.n
        self._check_buffers((("in0", in0), ("in1", in1), ("out0", out0), ("out1", out1)), dist, True)
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

    def execute_host(self, in0, out0, in1=None, out1=None,
                     direction: int = FORWARD, dist: Optional[int] = None) -> None:
        """Host fp32 buffers (numpy or pinned CPU tensors); pipelined H2D/compute/D2H."""
        if dist is None:
            dist = self.n
        self._check_buffers((("in0", in0), ("in1", in1), ("out0", out0), ("out1", out1)), dist, False)
        _check(lib.fftgen_execute_host(self._h, direction, _ptr(in0), _ptr(in1), _ptr(out0), _ptr(out1),
                                       int(dist)))

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

    def group_twiddles(self, group: int, which: int) -> np.ndarray:
        """Device twiddle table of a four-step group (0: Q, 1: P) as complex64."""
        cnt = int(lib.fftgen_plan_group_twiddles(self._h, group, which, None, 0))
        if cnt < 0:
            _check(5)
        out = np.empty(max(cnt, 0), dtype=np.complex64)
        if cnt:
            lib.fftgen_plan_group_twiddles(self._h, group, which, out.ctypes.data, cnt)
        return out

    def scratch_bytes(self) -> int:
        return int(lib.fftgen_plan_scratch_bytes(self._h))


TEXTS = {"formula": 0, "ir": 1, "loops": 2, "radices": 3}


def program_text(cfg: PipelineConfig, what: str = "formula") -> str:
    """Host-only program text of a config (no device): "formula"
    (print_formula, formula.cpp:104-146), "ir" (print_pipeline), "loops" (the
    sm_100a pass / group program) or "radices"."""
    c = _to_config(cfg)
    buf = C.create_string_buffer(1 << 22)
    _check(lib.fftgen_program_text(C.byref(c), TEXTS[what], buf, len(buf)))
    return buf.value.decode()


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
    import torch
    if block.device.type != "cuda":
        raise ExecError(f"twiddle_multiply needs a CUDA tensor, got {block.device}")
    if block.dtype == torch.complex64:
        if block.dim() != 2 or block.stride(1) != 1:
            raise ExecError("complex64 block must be 2-D with unit column stride")
        ld = block.stride(0)
    elif block.dtype == torch.float32:
        if block.dim() != 3 or block.shape[2] != 2 or block.stride(2) != 1 or block.stride(1) != 2 \
                or block.stride(0) % 2:
            raise ExecError("float32 block must be (rows, cols, 2) with interleaved (re, im) pairs")
        ld = block.stride(0) // 2
    else:
        raise ExecError(f"twiddle_multiply takes complex64 or float32 (rows, cols, 2), got {block.dtype}")
    rows, cols = block.shape[0], block.shape[1]
    if stream is None:
        stream = torch.cuda.current_stream(block.device).cuda_stream
    elif hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    _check(lib.fftgen_twiddle_multiply(direction, _ptr(block), rows, cols, ld, row_offset, col_offset, n,
                                       int(stream)))


def seeded_input(n: int, batch: int, layout: str = "interleaved", seed0: int = 1, device: int = 0,
                 dist: Optional[int] = None, stream=None):
    """The reference's seeded_input (verify.cpp:55-78) for `batch` transforms
    (seeds seed0 .. seed0+batch-1), generated on the device in fp32: a
    (batch, dist, 2) float32 tensor (interleaved) or a pair of (batch, dist)
    planes (split)."""
    import torch
    dist = n if dist is None else dist
    dev = torch.device("cuda", device)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    elif hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    if layout == "split":
        re = torch.empty(batch, dist, dtype=torch.float32, device=dev)
        im = torch.empty_like(re)
        _check(lib.fftgen_seeded_input(1, n, batch, seed0, _ptr(re), _ptr(im), dist, device, int(stream)))
        return re, im
    x = torch.empty(batch, dist, 2, dtype=torch.float32, device=dev)
    _check(lib.fftgen_seeded_input(0, n, batch, seed0, _ptr(x), None, dist, device, int(stream)))
    return x


class DistPlan:
    """One rank's share of a distributed n-point transform (fftgen_dist_plan):
    the P-point butterfly + D^N twiddle, the local n/world-point plan and the
    stride-world unpack (include/fftgen_b200.h, "distributed four-step").
    Buffers are CUDA complex64 (or float32 (..., 2)) blocks of n/world
    elements; the exchanges between the stages are the caller's
    (distributed.DistributedFFT)."""

    def __init__(self, n: int, world: int, rank: int, device: int = 0):
        h = C.c_void_p()
        _check(lib.fftgen_dist_plan_create(C.byref(h), int(n), int(world), int(rank), int(device)))
        self._h = h
        self.n, self.world, self.rank, self.device = int(n), int(world), int(rank), int(device)
        self.block = int(lib.fftgen_dist_block_elems(h))
        self.chunk = int(lib.fftgen_dist_chunk_elems(h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.fftgen_dist_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _buf(self, name, a):
        import torch
        if not hasattr(a, "data_ptr") or a.device.type != "cuda" or a.device.index != self.device:
            raise ExecError(f"{name} must be a CUDA tensor on cuda:{self.device}")
        if a.dtype not in (torch.complex64, torch.float32) or not a.is_contiguous():
            raise ExecError(f"{name} must be a contiguous complex64 / float32 tensor")
        elems = a.numel() if a.dtype == torch.complex64 else a.numel() // 2
        if elems != self.block:
            raise DimensionError(f"{name} holds {elems} elements, the rank's block is {self.block}")
        return _ptr(a)

    @staticmethod
    def _stream(stream, dev):
        import torch
        if stream is None:
            return torch.cuda.current_stream(dev).cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    def butterfly(self, recv, send, direction: int = FORWARD, stream=None) -> None:
        _check(lib.fftgen_dist_butterfly(self._h, direction, self._buf("recv", recv), self._buf("send", send),
                                         self._stream(stream, self.device)))

    def local(self, inp, out, direction: int = FORWARD, stream=None) -> None:
        _check(lib.fftgen_dist_local(self._h, direction, self._buf("in", inp), self._buf("out", out),
                                     self._stream(stream, self.device)))

    def unpack(self, recv, out, stream=None) -> None:
        _check(lib.fftgen_dist_unpack(self._h, self._buf("recv", recv), self._buf("out", out),
                                      self._stream(stream, self.device)))

    # ---- peer-memory transport (exchanges fused into the kernels) --------
    def _table(self, name, blocks):
        if len(blocks) != self.world:
            raise DimensionError(f"{name}: {len(blocks)} blocks for world {self.world}")
        ptrs = [int(b) if isinstance(b, int) else self._buf(name, b) for b in blocks]
        return (C.c_void_p * self.world)(*ptrs)

    def butterfly_peers(self, in_blocks, recv_blocks, direction: int = FORWARD, stream=None) -> None:
        """Exchange 1 + butterfly + exchange 2 in one kernel: in_blocks[r] /
        recv_blocks[r] are rank r's input / receive blocks (tensors on this
        device, or raw peer-mapped addresses)."""
        _check(lib.fftgen_dist_butterfly_peers(self._h, direction, self._table("in", in_blocks),
                                               self._table("recv", recv_blocks), self._stream(stream, self.device)))

    def unpack_peers(self, z_blocks, out, stream=None) -> None:
        """Exchange 3 + unpack in one kernel: pulls slot `rank` of every rank's
        local-result block z_blocks[q] into this rank's output."""
        _check(lib.fftgen_dist_unpack_peers(self._h, self._table("z", z_blocks), self._buf("out", out),
                                            self._stream(stream, self.device)))

    def describe_local(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        _check(lib.fftgen_plan_describe(lib.fftgen_dist_local_plan(self._h), buf, len(buf)))
        return buf.value.decode()

    def local_launches(self) -> int:
        return int(lib.fftgen_plan_launches(lib.fftgen_dist_local_plan(self._h)))


def flops(n: int, batch: int = 1) -> float:
    """5 N log2 N per transform (verify.cpp:48-51)."""
    return 5.0 * n * np.log2(n) * batch if n > 1 else 0.0
