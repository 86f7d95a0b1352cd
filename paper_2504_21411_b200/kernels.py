"""ctypes bindings to libgalv_b200.so (the C ABI in include/galv.h).

Thin, typed wrappers taking torch CUDA tensors: they pass raw device pointers,
sizes and the *current* CUDA stream, and raise ``RuntimeError`` with the
library's thread-local message on a non-zero status.  There is deliberately no
fallback: if the shared library is missing or the tensors are not on a CUDA
device the call fails loudly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
import os
from pathlib import Path

import torch

LIB_PATH = Path(os.environ["GALV_LIB"]) if os.environ.get("GALV_LIB") else Path(__file__).resolve().parent / "libgalv_b200.so"
F32, BF16 = 0, 1
_DT = {torch.float32: F32, torch.bfloat16: BF16}

_lib = None

_P, _I64, _I32, _F = C.c_void_p, C.c_int64, C.c_int32, C.c_float
_SIGS = {
    "galv_abi_version": ([], _I32),
    "galv_last_error": ([], C.c_char_p),
    "galv_device_info": ([_P, _P, _P], _I32),
    "galv_gemm": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _F, _I32,
                   _I32, _I32, _I32, _P], _I32),
    "galv_gemm_splits": ([_I64, _I64, _I64], _I32),
    "galv_gemm_splitk": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _F,
                          _I32, _I32, _I32, _I32, _P, _I64, _P], _I32),
    "galv_gemm_batched": ([_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                           _I64, _I32, _I32, _F, _I32, _I32, _I32, _P], _I32),
    "galv_gemm_rs": ([_P, _P, _P, _I64, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32,
                      _P], _I32),
    "galv_tp_signal_reduce": ([_P, _I32, _I32, C.c_uint32, _P, _P, _I64, _I32, _P], _I32),
    "galv_tp_allgather": ([_P, _P, _P, _I32, _I32, C.c_uint32, _I64, _P], _I32),
    "galv_comm_unique_id": ([_P], _I32),
    "galv_comm_init": ([_P, _I32, _I32, C.POINTER(C.c_void_p)], _I32),
    "galv_comm_split": ([_P, _I32, _I32, C.POINTER(C.c_void_p)], _I32),
    "galv_comm_destroy": ([_P], _I32),
    "galv_all_reduce": ([_P, _P, _P, _I64, _I32, _P], _I32),
    "galv_reduce_scatter": ([_P, _P, _P, _I64, _I32, _P], _I32),
    "galv_all_gather": ([_P, _P, _P, _I64, _I32, _P], _I32),
    "galv_sendrecv": ([_P, _P, _I64, _I32, _P, _I64, _I32, _P], _I32),
    "galv_nvl_signal": ([_P, _I32, _I32, C.c_uint32, _P], _I32),
    "galv_nvl_wait": ([_P, _I32, C.c_uint32, _P], _I32),
    "galv_dp_reduce": ([_P, _P, _I32, _I64, _P, _I32, _P, _P, _I64, _I32, _P], _I32),
    "galv_adamw_bcast": ([_P, _P, _P, _P, _P, _P, _I32, _I64, _I64, _F, _F, _F, _F, _F, _F,
                          _I64, _I32, _P], _I32),
    "galv_attn_fwd": ([_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _F, _I32,
                       _I32, _P], _I32),
    "galv_attn_bwd_workspace": ([_I64, _I64, _I64, _I64, _I32], _I64),
    "galv_gemm_splitk_workspace": ([_I64, _I64, _I64], _I64),
    "galv_colsum_workspace": ([_I64, _I64, _I32], _I64),
    "galv_attn_bwd": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64,
                       _I64, _F, _I32, _I32, _P, _P], _I32),
    "galv_attn_bwd_rope": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64,
                            _I64, _I64, _F, _I32, _P, _I32, _I32, _P, _P], _I32),
    "galv_attn_fwd_dropout": ([_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _F,
                               _I32, _F, C.c_uint64, C.c_uint64, _I64, _I64, _I64, _I32, _P],
                              _I32),
    "galv_attn_bwd_dropout": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64,
                               _I64, _I64, _F, _I32, _F, C.c_uint64, C.c_uint64, _I64, _I64,
                               _I64, _P, _I32, _I32, _P, _P], _I32),
    "galv_dropout_mask": ([_P, _I64, _I64, _I64, _F, C.c_uint64, C.c_uint64, _I64, _I64, _I64,
                           _P], _I32),
    "galv_rmsnorm_fwd": ([_P, _P, _P, _P, _P, _P, _I64, _I64, _F, _I32, _P], _I32),
    "galv_rmsnorm_bwd": ([_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I32, _P, _P], _I32),
    "galv_layernorm_fwd": ([_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _F, _I32, _P], _I32),
    "galv_layernorm_bwd": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I32, _P, _P],
                           _I32),
    "galv_norm_bwd_workspace": ([_I64, _I64], _I64),
    "galv_rope": ([_P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _F, _I32, _I32, _P], _I32),
    "galv_rope_table": ([_P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _P], _I32),
    "galv_swiglu_fwd": ([_P, _P, _I64, _I64, _I32, _P], _I32),
    "galv_swiglu_bwd": ([_P, _P, _P, _I64, _I64, _I32, _P], _I32),
    "galv_swiglu_bwd_strided": ([_P, _P, _I64, _P, _I64, _I64, _P], _I32),
    "galv_gemm_swiglu_fwd": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P],
                             _I32),
    "galv_gemm_swiglu_bwd": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P],
                             _I32),
    "galv_gemm_bias_gelu_fwd": ([_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                                 _I32, _P], _I32),
    "galv_gemm_bias_gelu_bwd": ([_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                                 _I32, _P], _I32),
    "galv_bias_gelu_fwd": ([_P, _P, _P, _I64, _I64, _I32, _P], _I32),
    "galv_bias_gelu_bwd": ([_P, _P, _P, _P, _I64, _I64, _I32, _P], _I32),
    "galv_bias_gelu_bwd_colsum": ([_P, _P, _P, _P, _P, _I64, _I64, _I32, _P], _I32),
    "galv_gemm_rope_qkv": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                            _P], _I32),
    "galv_bias_add": ([_P, _P, _I64, _I64, _I32, _P], _I32),
    "galv_colsum": ([_P, _P, _I64, _I64, _I32, _I32, _P, _P], _I32),
    "galv_embed_fwd": ([_P, _P, _P, _I64, _I64, _I64, _I64, _I32, _P], _I32),
    "galv_embed_bwd": ([_P, _P, _P, _I64, _I64, _I64, _I64, _I32, _P], _I32),
    "galv_embed_bwd_sorted": ([_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I32, _I32, _P], _I32),
    "galv_xent": ([_P, _P, _P, _P, _P, _I64, _I64, _I64, _F, _I64, _I32, _I32, _P], _I32),
    "galv_adamw": ([_P, _P, _P, _P, _P, _I64, _F, _F, _F, _F, _F, _F, _I64, _I32, _I32, _P],
                   _I32),
    "galv_gather_rows": ([_P, _P, _P, _I64, _I64, _P], _I32),
    "galv_scatter_rows": ([_P, _P, _P, _I64, _I64, _P], _I32),
    "galv_axpby": ([_P, _P, _I64, _F, _F, _I32, _I32, _P], _I32),
    "galv_sumsq": ([_P, _I64, _P, _I32, _P], _I32),
}
EXPORTED = tuple(_SIGS)


def load_library(path: str | os.PathLike | None = None):
    """Load (once) and type the C ABI; raises if the library or a symbol is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(f"{p} not built: run `python -m paper_2504_21411_b200.build` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    missing = []
    for name, (args, res) in _SIGS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.argtypes = args
        fn.restype = res
    lib.galv_missing = tuple(missing)
    if lib.galv_abi_version() != 1:
        raise RuntimeError("libgalv_b200 ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


# kernels launched per C-ABI call (for the bench's gpu_launches count); calls whose count
# depends on their arguments pass it to _call(launches=...) instead
KERNELS_PER_CALL = {"galv_attn_bwd": 3, "galv_tp_signal_reduce": 2, "galv_tp_allgather": 2}


class KernelStats:
    """Launch counter + optional CUDA-event timing of every GEMM (bench instrumentation)."""

    def __init__(self, time_gemm: bool = False):
        self.calls: dict = {}
        self.extra_launches = 0       # calls that reported their own launch count
        self.time_gemm = time_gemm
        self.gemm_events: list = []   # (flops, start_event, end_event, shape)

    @property
    def launches(self) -> int:
        return self.extra_launches + sum(n * KERNELS_PER_CALL.get(k, 1)
                                         for k, n in self.calls.items())

    def gemm_summary(self) -> dict:
        torch.cuda.synchronize()
        flops = sum(f for f, _, _, _ in self.gemm_events)
        ms = sum(a.elapsed_time(b) for _, a, b, _ in self.gemm_events)
        n = len(self.gemm_events)
        return {"launches": n, "flops": flops, "ms": ms,
                "tflops": flops / (ms * 1e-3) / 1e12 if ms else 0.0}


_stats: KernelStats | None = None


def start_stats(time_gemm: bool = False) -> KernelStats:
    global _stats
    _stats = KernelStats(time_gemm)
    return _stats


def stop_stats() -> KernelStats | None:
    global _stats
    s, _stats = _stats, None
    return s


def _call(name: str, *args, launches: int | None = None) -> None:
    if _stats is not None:
        if launches is None:
            _stats.calls[name] = _stats.calls.get(name, 0) + 1
        else:
            _stats.extra_launches += launches
    rc = getattr(load_library(), name)(*args)
    if rc != 0:
        msg = load_library().galv_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed (status {rc}): {msg}")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise RuntimeError("galv kernels need CUDA tensors (no CPU fallback)")
    return t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def dtype_code(dt) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise RuntimeError(f"unsupported dtype {dt}") from None


# ---------------------------------------------------------------------------- GEMM


_SPLITS: dict = {}


def _gemm_splits(M, N, K) -> int:
    key = (M, N, K)
    if key not in _SPLITS:
        _SPLITS[key] = int(load_library().galv_gemm_splits(M, N, K))
    return _SPLITS[key]


def gemm(a, b, out=None, *, trans_a=False, trans_b=False, alpha=1.0, accumulate=False,
         bias=None, out_dtype=None):
    """out[M,N] (+)= alpha * op(a) @ op(b) (+ bias).

    op(a): a is [M,K] (trans_a False) or [K,M] (True); op(b): b is [K,N] (trans_b
    False) or [N,K] (True, the nn.Linear weight layout).  Inputs must have unit
    stride in their last dim; leading dims are taken from stride(0).
    """
    if a.dim() != 2 or b.dim() != 2:
        raise RuntimeError("gemm expects 2-D operands")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise RuntimeError("gemm operands need a contiguous last dim")
    M, K = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    N, K2 = (b.shape[0], b.shape[1]) if trans_b else (b.shape[1], b.shape[0])
    if K != K2:
        raise RuntimeError(f"gemm K mismatch {K} vs {K2}")
    if a.dtype != b.dtype:
        raise RuntimeError("gemm operands must share a dtype")
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=out_dtype or a.dtype)
    if out.shape != (M, N) or out.stride(1) != 1:
        raise RuntimeError("bad gemm output")
    timed = _stats is not None and _stats.time_gemm
    if timed:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    splits = _gemm_splits(M, N, K) if a.dtype == torch.bfloat16 else 1
    if splits > 1:  # narrow output, long K: K-split units + one fp32 reduction pass
        nbytes = int(load_library().galv_gemm_splitk_workspace(M, N, K))
        ws = torch.empty(nbytes // 4, device=a.device, dtype=torch.float32)
        _call("galv_gemm_splitk", _ptr(a), _ptr(b), _ptr(out), _ptr(bias), M, N, K,
              a.stride(0), b.stride(0), out.stride(0), int(trans_a), int(trans_b),
              float(alpha), int(accumulate), dtype_code(out.dtype),
              dtype_code(bias.dtype) if bias is not None else F32, splits, _ptr(ws),
              ws.numel() * 4, _stream())
    else:
        _call("galv_gemm", _ptr(a), _ptr(b), _ptr(out), _ptr(bias), M, N, K, a.stride(0),
              b.stride(0), out.stride(0), int(trans_a), int(trans_b), float(alpha),
              int(accumulate), dtype_code(a.dtype), dtype_code(out.dtype),
              dtype_code(bias.dtype) if bias is not None else F32, _stream())
    if timed:
        ev1.record()
        _stats.gemm_events.append((2.0 * M * N * K, ev0, ev1, (M, N, K)))
    return out


def _timed_call(flops, shape, name, *args):
    timed = _stats is not None and _stats.time_gemm
    if timed:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    _call(name, *args)
    if timed:
        ev1.record()
        _stats.gemm_events.append((flops, ev0, ev1, shape))


def _bf16_rows(*ts):
    for t in ts:
        if t.dtype != torch.bfloat16 or t.dim() != 2 or t.stride(1) != 1:
            raise RuntimeError("fused SwiGLU GEMMs take bf16 2-D row-major tensors")


def gemm_swiglu_fwd(x, w_gu, gu=None, h=None):
    """gu = x @ w_gu^T ([T, 2F], gate then up) and h = silu(gate) * up ([T, F]), the
    activation fused into the GEMM epilogue (galv_gemm_swiglu_fwd)."""
    _bf16_rows(x, w_gu)
    T, Kd = x.shape
    F = w_gu.shape[0] // 2
    if w_gu.shape != (2 * F, Kd):
        raise RuntimeError("gate_up weight must be [2F, K]")
    gu = torch.empty(T, 2 * F, device=x.device, dtype=x.dtype) if gu is None else gu
    h = torch.empty(T, F, device=x.device, dtype=x.dtype) if h is None else h
    _timed_call(2.0 * T * 2 * F * Kd, (T, 2 * F, Kd), "galv_gemm_swiglu_fwd", _ptr(x),
                _ptr(w_gu), _ptr(gu), _ptr(h), T, F, Kd, x.stride(0), w_gu.stride(0),
                gu.stride(0), h.stride(0), _stream())
    return gu, h


def gemm_rope_qkv(x, w_qkv, seq_len, n_rot, *, theta=10000.0, out=None):
    """qkv = x @ w_qkv^T with RoPE (head_dim 128) applied to the first n_rot columns (the q
    and k heads) in the GEMM epilogue (galv_gemm_rope_qkv)."""
    _bf16_rows(x, w_qkv)
    T, Kd = x.shape
    N = w_qkv.shape[0]
    if w_qkv.shape[1] != Kd:
        raise RuntimeError("gemm_rope_qkv shape mismatch")
    out = torch.empty(T, N, device=x.device, dtype=x.dtype) if out is None else out
    table = rope_table(seq_len, 128, theta, x.device)
    _timed_call(2.0 * T * N * Kd, (T, N, Kd), "galv_gemm_rope_qkv", _ptr(x), _ptr(w_qkv),
                _ptr(out), _ptr(table), T, N, Kd, x.stride(0), w_qkv.stride(0), out.stride(0),
                n_rot, seq_len, _stream())
    return out


def gemm_swiglu_bwd(dy, w_down, gu, dgu=None):
    """d(gate|up) = swiglu_bwd(gu, dy @ w_down) with w_down [K, F] (the down projection's
    nn.Linear weight); the SwiGLU backward runs in the dgrad epilogue."""
    _bf16_rows(dy, w_down, gu)
    T, Kd = dy.shape
    F = w_down.shape[1]
    if w_down.shape[0] != Kd or gu.shape != (T, 2 * F):
        raise RuntimeError("gemm_swiglu_bwd shape mismatch")
    dgu = torch.empty_like(gu) if dgu is None else dgu
    _timed_call(2.0 * T * F * Kd, (T, F, Kd), "galv_gemm_swiglu_bwd", _ptr(dy), _ptr(w_down),
                _ptr(gu), _ptr(dgu), T, F, Kd, dy.stride(0), w_down.stride(0), gu.stride(0),
                dgu.stride(0), _stream())
    return dgu


def gemm_bias_gelu_fwd(x, w1, bias, pre=None, act=None):
    """pre = x @ w1^T and act = gelu_tanh(pre + bias), GeLU in the GEMM epilogue."""
    _bf16_rows(x, w1)
    T, Kd = x.shape
    F = w1.shape[0]
    if w1.shape[1] != Kd:
        raise RuntimeError("fc1 weight must be [F, K]")
    pre = torch.empty(T, F, device=x.device, dtype=x.dtype) if pre is None else pre
    act = torch.empty(T, F, device=x.device, dtype=x.dtype) if act is None else act
    _timed_call(2.0 * T * F * Kd, (T, F, Kd), "galv_gemm_bias_gelu_fwd", _ptr(x), _ptr(w1),
                _ptr(bias), _ptr(pre), _ptr(act), T, F, Kd, x.stride(0), w1.stride(0),
                pre.stride(0), act.stride(0), dtype_code(bias.dtype) if bias is not None else BF16,
                _stream())
    return pre, act


def gemm_bias_gelu_bwd(dy, w2, pre, bias, dpre=None):
    """dpre = (dy @ w2) * gelu_tanh'(pre + bias), w2 [K, F] (fc2's nn.Linear weight)."""
    _bf16_rows(dy, w2, pre)
    T, Kd = dy.shape
    F = w2.shape[1]
    if w2.shape[0] != Kd or pre.shape != (T, F):
        raise RuntimeError("gemm_bias_gelu_bwd shape mismatch")
    dpre = torch.empty_like(pre) if dpre is None else dpre
    _timed_call(2.0 * T * F * Kd, (T, F, Kd), "galv_gemm_bias_gelu_bwd", _ptr(dy), _ptr(w2),
                _ptr(pre), _ptr(bias), _ptr(dpre), T, F, Kd, dy.stride(0), w2.stride(0),
                pre.stride(0), dpre.stride(0),
                dtype_code(bias.dtype) if bias is not None else BF16, _stream())
    return dpre


def gemm_batched(a, b, out, *, trans_a=False, trans_b=False, alpha=1.0, accumulate=False):
    """Strided batched GEMM over the leading dim of 3-D operands."""
    Bt = a.shape[0]
    M, K = (a.shape[2], a.shape[1]) if trans_a else (a.shape[1], a.shape[2])
    N = b.shape[1] if trans_b else b.shape[2]
    _call("galv_gemm_batched", _ptr(a), _ptr(b), _ptr(out), Bt, a.stride(0), b.stride(0),
          out.stride(0), M, N, K, a.stride(1), b.stride(1), out.stride(1), int(trans_a),
          int(trans_b), float(alpha), int(accumulate), dtype_code(a.dtype),
          dtype_code(out.dtype), _stream())
    return out


# ---------------------------------------------------------------------------- attention


def _attn_geometry(q, o):
    # q/k/v: [B, S, H, D] views (possibly strided slices of a fused qkv buffer)
    B, S, H, D = q.shape
    if q.stride(3) != 1 or o.stride(3) != 1:
        raise RuntimeError("attention needs unit stride in head_dim")
    if q.stride(0) != S * q.stride(1) or o.stride(0) != S * o.stride(1):
        raise RuntimeError("attention needs [B, S] token-major packing")
    if o.stride(2) != q.stride(2):
        raise RuntimeError("q and o must share the head stride")
    return B, S, H, D, q.stride(1), q.stride(2), o.stride(1)


@dataclass(frozen=True)
class Dropout:
    """Attention-probability dropout of one call (csrc/dropout.cuh): probability p, Philox
    seed, per-call counter offset, and where this call's (b, h) sit in the global
    batch / head grid (b0, h0, H_total) so the mask is independent of the sharding."""
    p: float
    seed: int
    offset: int
    b0: int = 0
    h0: int = 0
    H_total: int = 0

    def args(self, H):
        return (float(self.p), int(self.seed) & 0xFFFFFFFFFFFFFFFF,
                int(self.offset) & 0xFFFFFFFFFFFFFFFF, int(self.b0), int(self.h0),
                int(self.H_total or H))


def attn_fwd(q, k, v, o, lse, *, scale, causal=True, dropout: Dropout | None = None):
    B, S, H, D, st, sh, ost = _attn_geometry(q, o)
    if k.stride() != q.stride() or v.stride() != q.stride():
        raise RuntimeError("q, k, v must share strides")
    if dropout is not None and dropout.p > 0:
        _call("galv_attn_fwd_dropout", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), B, S, H,
              D, st, sh, ost, float(scale), int(causal), *dropout.args(H), dtype_code(q.dtype),
              _stream())
        return
    _call("galv_attn_fwd", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), B, S, H, D, st, sh,
          ost, float(scale), int(causal), dtype_code(q.dtype), _stream())


def dropout_mask(B, S, H, dropout: Dropout, device="cuda"):
    """uint8 [B, H, S, S] keep mask the attention kernels apply for `dropout`."""
    m = torch.empty(B, H, S, S, dtype=torch.uint8, device=device)
    _call("galv_dropout_mask", _ptr(m), B, S, H, *dropout.args(H), _stream())
    return m


def attn_bwd_workspace_bytes(B, S, H, D, dtype) -> int:
    return int(load_library().galv_attn_bwd_workspace(B, S, H, D, dtype_code(dtype)))


def attn_bwd(q, k, v, o, dout, lse, dq, dk, dv, *, scale, causal=True, workspace=None,
             rope_theta=None, rope_epilogue=None, dropout: Dropout | None = None):
    """rope_theta set: dq/dk come out with the inverse RoPE applied (galv_attn_bwd_rope);
    rope_epilogue True/False forces the store-epilogue / streaming-pass variant, None takes
    the library default."""
    B, S, H, D, st, sh, ost = _attn_geometry(q, o)
    if dout.stride() != o.stride() or dq.stride() != q.stride():
        raise RuntimeError("dout must match o's layout and dq/dk/dv q's layout")
    need = load_library().galv_attn_bwd_workspace(B, S, H, D, dtype_code(q.dtype))
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=q.device)
    if dropout is not None and dropout.p > 0:
        table = rope_table(S, D, rope_theta, q.device) if rope_theta is not None else None
        epi = -1 if rope_epilogue is None else int(bool(rope_epilogue))
        if table is None or epi > 0:
            n = 3
        else:
            n = 4 if dk.data_ptr() == dq.data_ptr() + H * sh * dq.element_size() else 5
        _call("galv_attn_bwd_dropout", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout),
              _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv), B, S, H, D, st, sh, ost, float(scale),
              int(causal), *dropout.args(H), _ptr(table), epi, dtype_code(q.dtype),
              _ptr(workspace), _stream(), launches=n)
        return
    if rope_theta is not None:
        table = rope_table(S, D, rope_theta, q.device)
        # 3 backward kernels; the streaming variant adds one inverse-RoPE launch over q|k
        # when dk directly follows dq's heads in memory, else one each
        if rope_epilogue:
            n = 3
        else:
            n = 4 if dk.data_ptr() == dq.data_ptr() + H * sh * dq.element_size() else 5
        _call("galv_attn_bwd_rope", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout), _ptr(lse),
              _ptr(dq), _ptr(dk), _ptr(dv), B, S, H, D, st, sh, ost, float(scale), int(causal),
              _ptr(table), -1 if rope_epilogue is None else int(bool(rope_epilogue)),
              dtype_code(q.dtype), _ptr(workspace), _stream(), launches=n)
        return
    _call("galv_attn_bwd", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout), _ptr(lse), _ptr(dq),
          _ptr(dk), _ptr(dv), B, S, H, D, st, sh, ost, float(scale), int(causal),
          dtype_code(q.dtype), _ptr(workspace), _stream())


# ---------------------------------------------------------------------------- norms


def rmsnorm_fwd(x, gamma, eps, *, residual=None, res_out=None):
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    y = torch.empty_like(x)
    rstd = torch.empty(rows, device=x.device, dtype=torch.float32)
    _call("galv_rmsnorm_fwd", _ptr(x), _ptr(residual), _ptr(res_out), _ptr(gamma), _ptr(y),
          _ptr(rstd), rows, cols, float(eps), dtype_code(x.dtype), _stream())
    return y, rstd


def rmsnorm_bwd(x, gamma, rstd, dy, dgamma_acc, *, dres=None, dx=None):
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    dx = torch.empty_like(x) if dx is None else dx
    _call("galv_rmsnorm_bwd", _ptr(x), _ptr(gamma), _ptr(rstd), _ptr(dy), _ptr(dres), _ptr(dx),
          _ptr(dgamma_acc), rows, cols, dtype_code(x.dtype), None, _stream())
    return dx


def layernorm_fwd(x, gamma, beta, eps, *, residual=None, res_out=None):
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=x.device, dtype=torch.float32)
    rstd = torch.empty(rows, device=x.device, dtype=torch.float32)
    _call("galv_layernorm_fwd", _ptr(x), _ptr(residual), _ptr(res_out), _ptr(gamma),
          _ptr(beta), _ptr(y), _ptr(mean), _ptr(rstd), rows, cols, float(eps),
          dtype_code(x.dtype), _stream())
    return y, mean, rstd


def layernorm_bwd(x, gamma, mean, rstd, dy, dgamma_acc, dbeta_acc, *, dres=None, dx=None):
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    dx = torch.empty_like(x) if dx is None else dx
    _call("galv_layernorm_bwd", _ptr(x), _ptr(gamma), _ptr(mean), _ptr(rstd), _ptr(dy),
          _ptr(dres), _ptr(dx), _ptr(dgamma_acc), _ptr(dbeta_acc), rows, cols,
          dtype_code(x.dtype), None, _stream())
    return dx


# ---------------------------------------------------------------------------- pointwise


_ROPE_TABLES: dict = {}


def rope_table(seq_len, head_dim, theta, device):
    """fp32 [2, S, D/2] cos/sin planes, computed like the CPU restatement (fp32)."""
    key = (seq_len, head_dim, float(theta), str(device))
    t = _ROPE_TABLES.get(key)
    if t is None:
        inv = 1.0 / theta ** (torch.arange(0, head_dim, 2, dtype=torch.float32) / head_dim)
        ang = torch.arange(seq_len, dtype=torch.float32)[:, None] * inv[None, :]
        t = torch.stack([ang.cos(), ang.sin()]).contiguous().to(device)
        _ROPE_TABLES[key] = t
    return t


def rope_(x, seq_len, *, theta=10000.0, inverse=False, pos0=0):
    """In place on a [T, H, D] view (T = B*S tokens, token-major)."""
    T, H, D = x.shape
    if x.stride(2) != 1:
        raise RuntimeError("rope needs unit stride in head_dim")
    table = rope_table(seq_len, D, theta, x.device)
    _call("galv_rope_table", _ptr(x), _ptr(table), T, seq_len, H, D, x.stride(0), x.stride(1),
          pos0, int(inverse), dtype_code(x.dtype), _stream())
    return x


def swiglu_fwd(gu, out=None):
    T, F2 = gu.shape
    out = torch.empty(T, F2 // 2, device=gu.device, dtype=gu.dtype) if out is None else out
    _call("galv_swiglu_fwd", _ptr(gu), _ptr(out), T, F2 // 2, dtype_code(gu.dtype), _stream())
    return out


def swiglu_bwd(gu, dh, dgu=None):
    T, F2 = gu.shape
    dgu = torch.empty_like(gu) if dgu is None else dgu
    _call("galv_swiglu_bwd", _ptr(gu), _ptr(dh), _ptr(dgu), T, F2 // 2, dtype_code(gu.dtype),
          _stream())
    return dgu


def bias_gelu_fwd(x, bias, out=None):
    T, F = x.shape
    out = torch.empty_like(x) if out is None else out
    _call("galv_bias_gelu_fwd", _ptr(x), _ptr(bias), _ptr(out), T, F, dtype_code(x.dtype),
          _stream())
    return out


def bias_gelu_bwd(x, bias, dy, dx=None):
    T, F = x.shape
    dx = torch.empty_like(x) if dx is None else dx
    _call("galv_bias_gelu_bwd", _ptr(x), _ptr(bias), _ptr(dy), _ptr(dx), T, F,
          dtype_code(x.dtype), _stream())
    return dx


def bias_gelu_bwd_colsum(x, bias, dy, dbias_acc, dx=None):
    """dx = dy * gelu'(x + bias) and dbias_acc += dx.sum(0) in one pass."""
    T, F = x.shape
    dx = torch.empty_like(x) if dx is None else dx
    _call("galv_bias_gelu_bwd_colsum", _ptr(x), _ptr(bias), _ptr(dy), _ptr(dx),
          _ptr(dbias_acc), T, F, dtype_code(x.dtype), _stream())
    return dx


def colsum(x, out, *, accumulate=True):
    rows, cols = x.shape
    _call("galv_colsum", _ptr(x), _ptr(out), rows, cols, int(accumulate), dtype_code(x.dtype),
          None, _stream())
    return out


def embed_fwd(ids, table, vocab_lo=0, out=None):
    T = ids.numel()
    V, Hd = table.shape
    out = torch.empty(T, Hd, device=table.device, dtype=table.dtype) if out is None else out
    _call("galv_embed_fwd", _ptr(ids), _ptr(table), _ptr(out), T, V, vocab_lo, Hd,
          dtype_code(table.dtype), _stream())
    return out


def embed_bwd(ids, dout, dtable_acc, vocab_lo=0):
    T = ids.numel()
    V, Hd = dtable_acc.shape
    _call("galv_embed_bwd", _ptr(ids), _ptr(dout), _ptr(dtable_acc), T, V, vocab_lo, Hd,
          dtype_code(dout.dtype), _stream())


def embed_bwd_sorted(ids, dout, grad, vocab_lo=0):
    """grad[V_local, h] (bf16 or fp32) += per-id sums of dout rows (deterministic)."""
    sorted_ids, order = torch.sort(ids.reshape(-1), stable=True)
    T = sorted_ids.numel()
    V, Hd = grad.shape
    _call("galv_embed_bwd_sorted", _ptr(sorted_ids), _ptr(order), _ptr(dout), _ptr(grad), T, V,
          vocab_lo, Hd, dtype_code(dout.dtype), dtype_code(grad.dtype), _stream())


def xent(logits, labels, stats, stage, *, loss=None, dlogits=None, vocab_lo=0, grad_scale=1.0,
         ignore_index=-100):
    T, V = logits.shape
    _call("galv_xent", _ptr(logits), _ptr(labels), _ptr(stats), _ptr(loss), _ptr(dlogits), T,
          V, vocab_lo, float(grad_scale), int(ignore_index), int(stage),
          dtype_code(logits.dtype), _stream())


def adamw(master, m, v, grad, param_out, *, lr, beta1, beta2, eps, weight_decay, step,
          grad_scale=1.0):
    n = master.numel()
    _call("galv_adamw", _ptr(master), _ptr(m), _ptr(v), _ptr(grad), _ptr(param_out), n,
          float(lr), float(beta1), float(beta2), float(eps), float(weight_decay),
          float(grad_scale), int(step), dtype_code(grad.dtype),
          dtype_code(param_out.dtype) if param_out is not None else F32, _stream())


def gather_rows(src, idx, dst):
    row_bytes = src.stride(0) * src.element_size()
    _call("galv_gather_rows", _ptr(src), _ptr(dst), _ptr(idx), idx.numel(), row_bytes,
          _stream())
    return dst


def scatter_rows(src, idx, dst):
    row_bytes = src.stride(0) * src.element_size()
    _call("galv_scatter_rows", _ptr(src), _ptr(dst), _ptr(idx), idx.numel(), row_bytes,
          _stream())
    return dst


def axpby(x, y, a, b):
    _call("galv_axpby", _ptr(x), _ptr(y), x.numel(), float(a), float(b), dtype_code(x.dtype),
          dtype_code(y.dtype), _stream())
    return y


def sumsq(x, out):
    _call("galv_sumsq", _ptr(x), x.numel(), _ptr(out), dtype_code(x.dtype), _stream())
    return out


def bias_add_(x, bias):
    T, F = x.shape
    _call("galv_bias_add", _ptr(x), _ptr(bias), T, F, dtype_code(x.dtype), _stream())
    return x


# ---------------------------------------------------------------------------- TP over NVLink


def gemm_rs(a, b, peer_ptrs, rows_per_rank, my_slot, *, trans_a=False, trans_b=False,
            ldc=None):
    """Row-parallel GEMM whose epilogue stores rows into the tp ranks' receive buffers."""
    M, K = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    N = b.shape[0] if trans_b else b.shape[1]
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise RuntimeError("gemm_rs is bf16-only")
    timed = _stats is not None and _stats.time_gemm
    if timed:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    _call("galv_gemm_rs", _ptr(a), _ptr(b), _ptr(peer_ptrs), rows_per_rank, my_slot, M, N, K,
          a.stride(0), b.stride(0), ldc if ldc is not None else N, int(trans_a), int(trans_b),
          _stream())
    if timed:
        ev1.record()
        _stats.gemm_events.append((2.0 * M * N * K, ev0, ev1, (M, N, K)))


# ---------------------------------------------------------------- NCCL through the C ABI
def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _call("galv_comm_unique_id", C.cast(buf, C.c_void_p))
    return buf.raw


def comm_init(unique_id: bytes, nranks: int, rank: int) -> int:
    """Opaque NCCL communicator handle (call on every rank with the same id)."""
    buf = C.create_string_buffer(unique_id, 128)
    out = C.c_void_p()
    _call("galv_comm_init", C.cast(buf, C.c_void_p), nranks, rank, C.byref(out))
    return out.value


def comm_split(comm: int, color: int, key: int) -> int:
    out = C.c_void_p()
    _call("galv_comm_split", comm, color, key, C.byref(out))
    return out.value


def comm_destroy(comm: int) -> None:
    _call("galv_comm_destroy", comm)


def comm_all_reduce(comm: int, send, recv=None):
    recv = send if recv is None else recv
    _call("galv_all_reduce", comm, _ptr(send), _ptr(recv), send.numel(),
          dtype_code(send.dtype), _stream())
    return recv


def comm_reduce_scatter(comm: int, send, recv):
    _call("galv_reduce_scatter", comm, _ptr(send), _ptr(recv), recv.numel(),
          dtype_code(send.dtype), _stream())
    return recv


def comm_all_gather(comm: int, send, recv):
    _call("galv_all_gather", comm, _ptr(send), _ptr(recv), send.numel(),
          dtype_code(send.dtype), _stream())
    return recv


def comm_sendrecv(comm: int, send, peer_send: int, recv, peer_recv: int):
    nb = lambda t: 0 if t is None else t.numel() * t.element_size()
    _call("galv_sendrecv", comm, _ptr(send), nb(send), peer_send, _ptr(recv), nb(recv),
          peer_recv, _stream())


def nvl_signal(flag_ptrs, me, t, epoch):
    """Raise this rank's flag (epoch) in every peer's flag array (one warp)."""
    _call("galv_nvl_signal", _ptr(flag_ptrs), me, t, epoch & 0xFFFFFFFF, _stream())


def nvl_wait(my_flags_addr: int, t, epoch):
    """Single-CTA wait until every source rank's flag in this rank's array reached epoch."""
    _call("galv_nvl_wait", my_flags_addr, t, epoch & 0xFFFFFFFF, _stream())


def dp_reduce(*, n, t, mc_src=None, peer_src=None, offset=0, out=None, accumulate=False,
              mc_dst=None, peer_dst=None, max_ctas=0):
    """out (+)= sum over the dp ranks of their [offset, offset+n) bf16 slice (NVSwitch
    multimem.ld_reduce at mc_src, else unicast loads via the peer_src pointer array); the
    reduced slice is optionally stored to every rank (mc_dst / peer_dst): an all-reduce."""
    _call("galv_dp_reduce", mc_src, _ptr(peer_src), t, offset, _ptr(out), int(accumulate),
          mc_dst, _ptr(peer_dst), n, max_ctas, _stream())


def adamw_bcast(master, m, v, grad, *, t, offset, mc_dst=None, peer_dst=None, lr, beta1,
                beta2, eps, weight_decay, step, grad_scale=1.0):
    """AdamW on this rank's shard; bf16 params stored to every dp rank (fused all-gather)."""
    _call("galv_adamw_bcast", _ptr(master), _ptr(m), _ptr(v), _ptr(grad), mc_dst,
          _ptr(peer_dst), t, offset, master.numel(), float(lr), float(beta1), float(beta2),
          float(eps), float(weight_decay), float(grad_scale), int(step),
          dtype_code(grad.dtype), _stream())


def tp_signal_reduce(flag_ptrs, me, t, epoch, recv, out):
    _call("galv_tp_signal_reduce", _ptr(flag_ptrs), me, t, epoch & 0xFFFFFFFF, _ptr(recv),
          _ptr(out), out.numel(), dtype_code(out.dtype), _stream())
    return out


def tp_allgather(src, dst_ptrs, flag_ptrs, me, t, epoch):
    _call("galv_tp_allgather", _ptr(src), _ptr(dst_ptrs), _ptr(flag_ptrs), me, t,
          epoch & 0xFFFFFFFF, src.numel() * src.element_size(), _stream())
