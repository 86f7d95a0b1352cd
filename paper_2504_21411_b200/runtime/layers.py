"""Decoder layers, embedding and LM head with explicit forward/backward on galv kernels.

Each layer realizes its ``ParallelStrategy`` (reference strategy.py:20-60):
  * tp: Megatron column-parallel QKV / fc1 / gate_up and row-parallel proj / fc2 / down
    (heads and FFN columns split over the contiguous tp group)
  * sp: the residual stream is token-sharded over the tp group; all-gather before the
    column GEMMs, reduce-scatter after the row GEMMs (same volume as the AR pair,
    costmodel.py:7-10)
  * dp / zero_stage: see params.ParamStore
  * recompute: forward keeps only the layer input; backward replays the forward
    (including its tp traffic, costmodel.py:122-126) and then runs backward.

Activations are 2-D [tokens, hidden] in token-major [b, s] order.  Tokens of a
microbatch are split into dp replicas (contiguous sample ranges) and, under sp, into
tp chunks of contiguous tokens (per-token ops do not care which tokens a rank owns;
attention runs on the gathered full sequences).
"""

from __future__ import annotations

import math

import torch

from .. import kernels as K
from . import comm
from .params import ParamStore

SMALL_SUFFIXES = ("norm.weight", "norm.bias", ".bias")


def _is_small(name: str) -> bool:
    return name.endswith(SMALL_SUFFIXES)


# ---------------------------------------------------------------------------- TP slicing


def tp_slice(cfg, name: str, full: torch.Tensor, tp: int, r: int) -> torch.Tensor:
    """Local shard of a logical tensor for tp rank r (Megatron layout)."""
    if tp == 1:
        return full
    leaf = name.split(".", 2)[-1] if name.startswith("layers.") else name
    h, f = cfg.hidden, cfg.ffn
    if leaf in ("qkv.weight", "qkv.bias"):
        hl = h // tp
        parts = [full[j * h + r * hl: j * h + (r + 1) * hl] for j in range(3)]
        return torch.cat(parts, 0)
    if leaf in ("fc1.weight", "fc1.bias"):
        fl = f // tp
        return full[r * fl:(r + 1) * fl]
    if leaf == "gate_up.weight":
        fl = f // tp
        return torch.cat([full[r * fl:(r + 1) * fl], full[f + r * fl: f + (r + 1) * fl]], 0)
    if leaf in ("proj.weight",):
        hl = h // tp
        return full[:, r * hl:(r + 1) * hl]
    if leaf in ("fc2.weight", "down.weight"):
        fl = f // tp
        return full[:, r * fl:(r + 1) * fl]
    if leaf in ("embed.weight", "lm_head.weight"):
        vl = cfg.vocab // tp
        return full[r * vl:(r + 1) * vl]
    return full  # norms, row-parallel output biases, positional embedding: replicated


def tp_unslice(cfg, name: str, parts: list) -> torch.Tensor:
    """Inverse of tp_slice over the tp ranks' shards (tests / checkpoint export)."""
    tp = len(parts)
    if tp == 1:
        return parts[0]
    leaf = name.split(".", 2)[-1] if name.startswith("layers.") else name
    if leaf in ("qkv.weight", "qkv.bias"):
        hl = cfg.hidden // tp
        return torch.cat([p[j * hl:(j + 1) * hl] for j in range(3) for p in parts], 0)
    if leaf == "gate_up.weight":
        fl = cfg.ffn // tp
        return torch.cat([p[:fl] for p in parts] + [p[fl:] for p in parts], 0)
    if leaf in ("fc1.weight", "fc1.bias", "embed.weight", "lm_head.weight"):
        return torch.cat(parts, 0)
    if leaf in ("proj.weight", "fc2.weight", "down.weight"):
        return torch.cat(parts, 1)
    return parts[0]


# ---------------------------------------------------------------------------- helpers


# Fused activation epilogues pay off once the GEMM mainloop (K = hidden) is long enough to
# hide them (scratch/gelu_bench.py, scratch/swiglu_bench.py on B200): forward from K >= 2048,
# the backward (which also streams the saved pre-activation) from K >= 4096.
FUSE_ACT_FWD_MIN_K = 2048
FUSE_ACT_BWD_MIN_K = 4096
# galv_attn_bwd_rope variant: None = library default (backward + one streaming inverse-RoPE
# pass), True = rotation in the dq/dk store epilogues
ROPE_BWD_EPILOGUE = None


def _fuse_fwd(x):
    return x.dtype == torch.bfloat16 and x.shape[1] >= FUSE_ACT_FWD_MIN_K


def _fuse_bwd(dy):
    return dy.dtype == torch.bfloat16 and dy.shape[1] >= FUSE_ACT_BWD_MIN_K


def _linear(x, w, out=None, bias=None):
    """x [T, K] @ w[N, K]^T (+bias) -> [T, N]."""
    return K.gemm(x, w, out, trans_b=True, bias=bias)


def _dgrad(dy, w, out=None):
    """dy [T, N] @ w [N, K] -> [T, K]."""
    return K.gemm(dy, w, out)


def _wgrad(dy, x, gw):
    """gw [N, K] += dy^T [N, T] @ x [T, K]."""
    K.gemm(dy, x, gw, trans_a=True, accumulate=True)


class _Ctx:
    __slots__ = ("saved", "x")

    def __init__(self):
        self.saved = None
        self.x = None


# ---------------------------------------------------------------------------- decoder layer


class DecoderLayer:
    def __init__(self, cfg, index: int, strategy, topo, *, dtype, grad_dtype, device):
        self.cfg, self.index, self.s = cfg, index, strategy
        self.dtype, self.device = dtype, device
        self.tpg = topo.tp(strategy.tp)
        self.dpg = topo.dp(strategy.tp)
        self.tp, self.tpr = strategy.tp, self.tpg.index
        # Ulysses: sp layers keep full weights in the group and shard only the sequence
        self.uly = bool(strategy.sp and strategy.tp > 1 and topo.hc.sp_mode == "ulysses")
        self.wtp, self.wtpr = (1, 0) if self.uly else (self.tp, self.tpr)
        h, f = cfg.hidden, cfg.ffn
        self.hl, self.fl = h // self.wtp, f // self.wtp       # GEMM widths
        self.Hl = cfg.heads // self.tp                        # attention heads per rank
        self.ahl = self.Hl * cfg.head_dim                     # attention width per rank
        from .init import layer_param_shapes
        shapes = layer_param_shapes(cfg)
        local = {}
        for n, shp in shapes.items():
            local[n] = tuple(tp_slice(cfg, n, torch.empty(shp, device="meta"), self.wtp,
                                      self.wtpr).shape)
        self.names = list(shapes)
        self.store = ParamStore([(n, local[n]) for n in self.names], dtype=dtype,
                                grad_dtype=grad_dtype, device=device, dp=self.dpg,
                                zero=strategy.zero_stage,
                                small_names=[n for n in self.names if _is_small(n)],
                                extra_allreduce=self.tpg if self.uly else None)
        # replicated params whose grads are token-partial under Megatron-SP
        self.tp_partial = [] if self.uly else [
            n for n in self.names if _is_small(n) and strategy.sp and
            n not in ("qkv.bias", "fc1.bias")]
        self._uly_idx = {}
        # Megatron-SP row GEMMs: reduce-scatter fused into the GEMM over NVLink peer memory
        self.peer = None
        if (self.tp > 1 and not self.uly and dtype == torch.bfloat16 and topo.distributed):
            from . import nvlink
            if nvlink.enabled() and (strategy.sp or nvlink.allreduce_enabled()):
                T = topo.hc.microbatch // strategy.dp * cfg.seq_len
                self.peer = nvlink.peer_buffers(self.tpg, T * max(cfg.hidden, 1) * 2, device)
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        # attention dropout (cfg.attn_dropout): Philox seed and the step counter the engine
        # advances per train_step; the counter offset is (step << 16) | layer index
        self.dropout_seed, self.dropout_step = 0, 0

    def param_prefix(self) -> str:
        return f"layers.{self.index}."

    # -------------------------------------------------------------- forward
    def _gather_seq(self, t):
        return comm.all_gather(t, self.tpg) if (self.s.sp and not self.uly) else t

    def _reduce_out(self, t):
        if self.tp == 1 or self.uly:
            return t
        if self.s.sp:
            return comm.reduce_scatter(t, self.tpg)
        return comm.all_reduce(t, self.tpg)

    def _row_gemm(self, x, w, *, trans_b, bias=None):
        """Row-parallel GEMM + tp reduction (fused NVLink reduce-scatter under Megatron-SP)."""
        if self.peer is not None and bias is None:
            if self.s.sp:
                return self.peer.gemm_rs(x, w, trans_b=trans_b)
            return self.peer.gemm_ar(x, w, trans_b=trans_b)
        y = K.gemm(x, w, trans_b=trans_b, bias=bias)
        return self._reduce_out(y)

    def _norm_fwd(self, x, w, prefix, residual=None):
        res_out = torch.empty_like(x) if residual is not None else None
        if self.cfg.arch == "gpt":
            y, mean, rstd = K.layernorm_fwd(x, w[prefix + ".weight"], w[prefix + ".bias"],
                                            self.cfg.norm_eps, residual=residual,
                                            res_out=res_out)
        else:
            y, rstd = K.rmsnorm_fwd(x, w[prefix + ".weight"], self.cfg.norm_eps,
                                    residual=residual, res_out=res_out)
            mean = None
        return y, (mean, rstd), res_out

    def _norm_bwd(self, x, w, stats, dy, prefix, sg, dres=None):
        mean, rstd = stats
        if self.cfg.arch == "gpt":
            return K.layernorm_bwd(x, w[prefix + ".weight"], mean, rstd, dy,
                                   sg[prefix + ".weight"], sg[prefix + ".bias"], dres=dres)
        return K.rmsnorm_bwd(x, w[prefix + ".weight"], rstd, dy, sg[prefix + ".weight"],
                             dres=dres)

    # ------------------------------------------------------------- Ulysses all-to-alls
    def _uly_maps(self, Tl):
        """Row-index maps (rows = one head vector) for the sequence<->head all-to-alls."""
        key = Tl
        if key not in self._uly_idx:
            u, H, Hl = self.tp, self.cfg.heads, self.Hl
            dev = self.device
            j = torch.arange(u).view(u, 1, 1, 1)
            t = torch.arange(Tl).view(1, Tl, 1, 1)
            p = torch.arange(3).view(1, 1, 3, 1)
            hh = torch.arange(Hl).view(1, 1, 1, Hl)
            # pack for qkv: local [Tl, 3, H] rows -> (dest j, t, p, hl)
            qkv_pack = (t * (3 * H) + p * H + j * Hl + hh).reshape(-1)
            jj = torch.arange(u).view(u, 1, 1)
            tt = torch.arange(Tl).view(1, Tl, 1)
            h2 = torch.arange(Hl).view(1, 1, Hl)
            # o: received (src r, t, hl) -> local [Tl, H] row t*H + r*Hl + hl
            o_unpack = (tt * H + jj * Hl + h2).reshape(-1)
            self._uly_idx[key] = (qkv_pack.to(dev), o_unpack.to(dev))
        return self._uly_idx[key]

    def _uly_qkv_to_heads(self, qkv_local):
        """[Tl, 3h] (all heads, local tokens) -> [T, 3*Hl*D] (local heads, all tokens)."""
        Tl, D = qkv_local.shape[0], self.cfg.head_dim
        pack, _ = self._uly_maps(Tl)
        rows = qkv_local.view(-1, D)
        send = torch.empty(pack.numel(), D, dtype=qkv_local.dtype, device=qkv_local.device)
        K.gather_rows(rows, pack, send)
        out = torch.empty(Tl * self.tp, 3 * self.ahl, dtype=qkv_local.dtype,
                          device=qkv_local.device)
        n = send.shape[0] // self.tp
        comm.all_to_all(out.view(-1, D), send, [n] * self.tp, [n] * self.tp, self.tpg)
        return out

    def _uly_heads_to_qkv(self, dqkv_full):
        """inverse of _uly_qkv_to_heads (gradient direction)."""
        T, D = dqkv_full.shape[0], self.cfg.head_dim
        Tl = T // self.tp
        pack, _ = self._uly_maps(Tl)
        recv = torch.empty(pack.numel(), D, dtype=dqkv_full.dtype, device=dqkv_full.device)
        n = recv.shape[0] // self.tp
        comm.all_to_all(recv, dqkv_full.view(-1, D), [n] * self.tp, [n] * self.tp, self.tpg)
        out = torch.empty(Tl, 3 * self.cfg.hidden, dtype=dqkv_full.dtype,
                          device=dqkv_full.device)
        K.scatter_rows(recv, pack, out.view(-1, D))
        return out

    def _uly_o_to_tokens(self, o_full):
        """[T, Hl*D] -> [Tl, h]: attention output back to the local tokens, all heads."""
        T, D = o_full.shape[0], self.cfg.head_dim
        Tl = T // self.tp
        _, unpack = self._uly_maps(Tl)
        recv = torch.empty(T * self.Hl, D, dtype=o_full.dtype, device=o_full.device)
        n = recv.shape[0] // self.tp
        comm.all_to_all(recv, o_full.view(-1, D), [n] * self.tp, [n] * self.tp, self.tpg)
        out = torch.empty(Tl, self.cfg.hidden, dtype=o_full.dtype, device=o_full.device)
        K.scatter_rows(recv, unpack, out.view(-1, D))
        return out

    def _uly_tokens_to_o(self, do_local):
        """inverse of _uly_o_to_tokens (gradient direction)."""
        Tl, D = do_local.shape[0], self.cfg.head_dim
        _, unpack = self._uly_maps(Tl)
        send = torch.empty(unpack.numel(), D, dtype=do_local.dtype, device=do_local.device)
        K.gather_rows(do_local.view(-1, D), unpack, send)
        out = torch.empty(Tl * self.tp, self.ahl, dtype=do_local.dtype, device=do_local.device)
        n = send.shape[0] // self.tp
        comm.all_to_all(out.view(-1, D), send, [n] * self.tp, [n] * self.tp, self.tpg)
        return out

    def _attn_views(self, qkv, B, S):
        hl, D = self.ahl, self.cfg.head_dim
        st = qkv.stride(0)
        base = qkv.storage_offset()
        mk = lambda j: qkv.as_strided((B, S, self.Hl, D), (S * st, st, D, 1), base + j * hl)
        return mk(0), mk(1), mk(2)

    def _dropout(self, b0: int):
        """Dropout of this layer's attention call: global sample b0 of its first sequence,
        global head h0 of its first head (tp / Ulysses ranks own contiguous head blocks)."""
        if self.cfg.attn_dropout <= 0:
            return None
        return K.Dropout(self.cfg.attn_dropout, self.dropout_seed,
                         (self.dropout_step << 16) | self.index, b0=b0, h0=self.tpr * self.Hl,
                         H_total=self.cfg.heads)

    def forward_impl(self, x, B, save: bool, keep_gathered: bool = False, b0: int = 0):
        """x: [T_in, h] in this layer's layout; B = samples in this dp replica.

        Under Megatron-SP the saved norm outputs are this rank's token shards (n1, n2),
        as the cost model counts them (replicated activations / tp, costmodel.py:162-175);
        the backward all-gathers them again, overlapped with its dgrad GEMMs (Megatron
        does the same).  A recompute replay (keep_gathered) keeps the gathered copies:
        only one layer's activations are alive then."""
        cfg = self.cfg
        S = cfg.seq_len
        flat = self.store.materialize()
        w = self.store.views(flat)
        gpt = cfg.arch == "gpt"
        n1, st1, _ = self._norm_fwd(x, w, "attn_norm")
        n1f = self._gather_seq(n1)
        T = n1f.shape[0]
        # Llama: RoPE on the q|k heads inside the QKV GEMM epilogue (Ulysses rotates after
        # its head all-to-all, so it keeps the standalone kernel)
        rope_fused = (not gpt and not self.uly and cfg.head_dim == 128
                      and n1f.dtype == torch.bfloat16)
        if rope_fused:
            qkv = K.gemm_rope_qkv(n1f, w["qkv.weight"], S, 2 * self.ahl, theta=cfg.rope_theta)
        else:
            qkv = _linear(n1f, w["qkv.weight"], bias=w["qkv.bias"] if gpt else None)
        if self.uly:
            qkv = self._uly_qkv_to_heads(qkv)
            T = qkv.shape[0]
        q, k, v = self._attn_views(qkv, B, S)
        if not gpt and not rope_fused:
            # q and k heads are adjacent in the qkv row ([q | k | v], ahl = Hl*D each):
            # one launch rotates all 2*Hl of them
            K.rope_(qkv.as_strided((T, 2 * self.Hl, cfg.head_dim),
                                   (qkv.stride(0), cfg.head_dim, 1), qkv.storage_offset()),
                    S, theta=cfg.rope_theta)
        o = torch.empty(T, self.ahl, device=x.device, dtype=x.dtype)
        lse = torch.empty(B, self.Hl, S, device=x.device, dtype=torch.float32)
        drop = self._dropout(b0)
        K.attn_fwd(q, k, v, o.view(B, S, self.Hl, cfg.head_dim), lse, scale=self.scale,
                   causal=True, dropout=drop)
        o_full = o
        if self.uly:
            o = self._uly_o_to_tokens(o_full)
        fuse_bias = gpt and self.wtp == 1
        a = self._row_gemm(o, w["proj.weight"], trans_b=True,
                           bias=w["proj.bias"] if fuse_bias else None)
        if gpt and not fuse_bias:
            K.bias_add_(a, w["proj.bias"])
        # h1 = x + a ; n2 = norm(h1)
        n2, st2, h1 = self._norm_fwd(a, w, "mlp_norm", residual=x)
        n2f = self._gather_seq(n2)
        if gpt:
            if _fuse_fwd(n2f):  # bias-GeLU fused into the fc1 GEMM epilogue
                f1, act = K.gemm_bias_gelu_fwd(n2f, w["fc1.weight"], w["fc1.bias"])
            else:
                f1 = _linear(n2f, w["fc1.weight"])       # pre-activation (bias in gelu)
                act = K.bias_gelu_fwd(f1, w["fc1.bias"])
            m = self._row_gemm(act, w["fc2.weight"], trans_b=True,
                               bias=w["fc2.bias"] if fuse_bias else None)
        else:
            if _fuse_fwd(n2f):  # SwiGLU fused into the gate|up GEMM epilogue
                gu, act = K.gemm_swiglu_fwd(n2f, w["gate_up.weight"])
            else:
                gu = _linear(n2f, w["gate_up.weight"])
                act = K.swiglu_fwd(gu)
            m = self._row_gemm(act, w["down.weight"], trans_b=True)
        if gpt and not fuse_bias:
            K.bias_add_(m, w["fc2.bias"])
        y = K.axpby(h1, m, 1.0, 1.0)
        if save:
            regather = self.s.sp and not self.uly and self.tp > 1 and not keep_gathered
            saved = dict(x=x, st1=st1, n1f=n1 if regather else n1f, qkv=qkv, o=o,
                         o_full=o_full, lse=lse, h1=h1, st2=st2,
                         n2f=n2 if regather else n2f, act=act, B=B, regather=regather,
                         drop=drop)
            saved["pre"] = f1 if gpt else gu
            return y, saved
        return y, None

    def forward(self, x, B, b0: int = 0):
        """b0: global index of this replica's first sample (attention-dropout coordinates)."""
        ctx = _Ctx()
        if self.s.recompute:
            y, _ = self.forward_impl(x, B, save=False, b0=b0)
            ctx.x, ctx.saved = (x, B, b0), None
        else:
            y, ctx.saved = self.forward_impl(x, B, save=True, b0=b0)
        self.store.release()
        return y, ctx

    # -------------------------------------------------------------- backward
    def backward(self, dy, ctx):
        cfg = self.cfg
        if ctx.saved is None:
            x, B, b0 = ctx.x
            _, sv = self.forward_impl(x, B, save=True, keep_gathered=True, b0=b0)
        else:
            sv = ctx.saved
        ctx.saved = ctx.x = None
        S = cfg.seq_len
        gpt = cfg.arch == "gpt"
        flat = self.store.materialize()
        w = self.store.views(flat)
        gflat = self.store.grad_target()
        gw = self.store.views(gflat)
        sg = self.store.small_grads()
        B = sv["B"]
        # ---- MLP
        dmf = self._gather_seq(dy)
        n2f = n2_work = n1f = n1_work = None
        if sv["regather"]:  # SP: re-gather the norm-2 output behind the dgrad GEMM
            n2f, n2_work = comm.all_gather_async(sv["n2f"], self.tpg)
        else:
            n2f = sv["n2f"]
        if gpt:
            K.colsum(dy, sg["fc2.bias"])
            if _fuse_bwd(dmf):  # GeLU bwd fused into the fc2 dgrad epilogue
                dpre = K.gemm_bias_gelu_bwd(dmf, w["fc2.weight"], sv["pre"], w["fc1.bias"])
            else:
                dact = _dgrad(dmf, w["fc2.weight"])
                # bias grad summed in the same pass over dpre
                dpre = K.bias_gelu_bwd_colsum(sv["pre"], w["fc1.bias"], dact, sg["fc1.bias"])
                del dact
            _wgrad(dmf, sv["act"], gw["fc2.weight"])
            if _fuse_bwd(dmf):
                K.colsum(dpre, sg["fc1.bias"])
            dn2 = self._row_gemm(dpre, w["fc1.weight"], trans_b=False)
            if n2_work is not None:
                n2_work.wait()
            _wgrad(dpre, n2f, gw["fc1.weight"])
        else:
            if _fuse_bwd(dmf):  # SwiGLU bwd fused into the down dgrad epilogue
                dpre = K.gemm_swiglu_bwd(dmf, w["down.weight"], sv["pre"])
            else:
                dact = _dgrad(dmf, w["down.weight"])
                dpre = K.swiglu_bwd(sv["pre"], dact)
                del dact
            _wgrad(dmf, sv["act"], gw["down.weight"])
            dn2 = self._row_gemm(dpre, w["gate_up.weight"], trans_b=False)
            if n2_work is not None:
                n2_work.wait()
            _wgrad(dpre, n2f, gw["gate_up.weight"])
        del dpre, dmf, n2f
        dh1 = self._norm_bwd(sv["h1"], w, sv["st2"], dn2, "mlp_norm", sg, dres=dy)
        del dn2
        # ---- attention
        daf = self._gather_seq(dh1)
        if sv["regather"]:  # norm-1 output, behind the attention backward
            n1f, n1_work = comm.all_gather_async(sv["n1f"], self.tpg)
        else:
            n1f = sv["n1f"]
        if gpt:
            K.colsum(dh1, sg["proj.bias"])
        do = _dgrad(daf, w["proj.weight"])
        _wgrad(daf, sv["o"], gw["proj.weight"])
        del daf
        if self.uly:
            do = self._uly_tokens_to_o(do)
        qkv = sv["qkv"]
        T = qkv.shape[0]
        dqkv = torch.empty_like(qkv)
        q, k, v = self._attn_views(qkv, B, S)
        dq, dk, dv = self._attn_views(dqkv, B, S)
        # transient (caching allocator): part of the measured backward working set, not a
        # per-layer resident buffer outside the cost model
        ws = torch.empty(K.attn_bwd_workspace_bytes(B, S, self.Hl, cfg.head_dim, qkv.dtype),
                         dtype=torch.uint8, device=qkv.device)
        # Llama, head_dim 128: dq / dk come back through the inverse RoPE of q / k in the
        # same C-ABI call (galv_attn_bwd_rope; its default variant is the streaming pass)
        rope_fused = not gpt and cfg.head_dim == 128 and qkv.dtype == torch.bfloat16
        K.attn_bwd(q, k, v, sv["o_full"].view(B, S, self.Hl, cfg.head_dim),
                   do.view(B, S, self.Hl, cfg.head_dim), sv["lse"], dq, dk, dv,
                   scale=self.scale, causal=True, workspace=ws,
                   rope_theta=cfg.rope_theta if rope_fused else None,
                   rope_epilogue=ROPE_BWD_EPILOGUE, dropout=sv["drop"])
        del do
        if not gpt and not rope_fused:
            K.rope_(dqkv.as_strided((T, 2 * self.Hl, cfg.head_dim),
                                    (dqkv.stride(0), cfg.head_dim, 1), dqkv.storage_offset()),
                    S, theta=cfg.rope_theta, inverse=True)
        if self.uly:
            dqkv = self._uly_heads_to_qkv(dqkv)
        if gpt:
            K.colsum(dqkv, sg["qkv.bias"])
        dn1 = self._row_gemm(dqkv, w["qkv.weight"], trans_b=False)
        if n1_work is not None:
            n1_work.wait()
        _wgrad(dqkv, n1f, gw["qkv.weight"])
        del dqkv, n1f
        dx = self._norm_bwd(sv["x"], w, sv["st1"], dn1, "attn_norm", sg, dres=dh1)
        self.store.release()
        self.store.finish_microbatch(gflat, self.tp_partial, self.tpg)
        return dx


# ---------------------------------------------------------------------------- embedding


class Embedding:
    """Vocab-parallel token embedding (+ learned positions for GPT) in layer 0's layout."""

    def __init__(self, cfg, strategy, topo, *, dtype, grad_dtype, device):
        self.cfg, self.s, self.dtype = cfg, strategy, dtype
        self.tpg, self.dpg = topo.tp(strategy.tp), topo.dp(strategy.tp)
        self.tp, self.tpr = strategy.tp, self.tpg.index
        self.vl = cfg.vocab // self.tp
        entries = [("embed.weight", (self.vl, cfg.hidden))]
        if cfg.arch == "gpt":
            entries.append(("pos_embed.weight", (cfg.seq_len, cfg.hidden)))
        # the tables follow layer 0's ZeRO stage: the cost model charges them to layer 0
        # (profiler.fold_embedding_head), so params / grads / optimizer state shard alike
        self.store = ParamStore(entries, dtype=dtype, grad_dtype=grad_dtype, device=device,
                                dp=self.dpg, zero=strategy.zero_stage)

    def forward(self, ids):
        """ids: [T_rep] int64 (this dp replica's tokens) -> [T_in, h] in layer-0 layout."""
        w = self.store.views(self.store.materialize())
        x = K.embed_fwd(ids, w["embed.weight"], vocab_lo=self.tpr * self.vl)
        if self.tp > 1:
            x = comm.reduce_scatter(x, self.tpg) if self.s.sp else comm.all_reduce(x, self.tpg)
        if self.cfg.arch == "gpt":
            S = self.cfg.seq_len
            T = x.shape[0]
            lo = self.tpr * T if (self.s.sp and self.tp > 1) else 0
            pos = w["pos_embed.weight"]
            rows = (torch.arange(lo, lo + T, device=x.device) % S)
            x.add_(pos.index_select(0, rows))
        self.store.release()
        return x

    def backward(self, ids, dx):
        cfg = self.cfg
        dxf = comm.all_gather(dx, self.tpg) if (self.s.sp and self.tp > 1) else dx
        gflat = self.store.grad_target()
        gw = self.store.views(gflat)
        # deterministic sorted segment-sum straight into the (bf16 or fp32) grad rows: no
        # fp32 [V, h] scratch table (it would sit outside the cost model's grad bytes)
        K.embed_bwd_sorted(ids, dxf, gw["embed.weight"], vocab_lo=self.tpr * self.vl)
        if cfg.arch == "gpt":
            S = cfg.seq_len
            T = dx.shape[0]
            lo = self.tpr * T if (self.s.sp and self.tp > 1) else 0
            rows = torch.arange(lo, lo + T, device=dx.device) % S
            acc = torch.zeros(S, cfg.hidden, dtype=torch.float32, device=dx.device)
            acc.index_add_(0, rows, dx.float())
            if self.s.sp and self.tp > 1:
                comm.all_reduce(acc, self.tpg)
            K.axpby(acc, gw["pos_embed.weight"], 1.0, 1.0)
        self.store.finish_microbatch(gflat)


# ---------------------------------------------------------------------------- head


# logits above HEAD_CHUNK_BYTES are processed in token chunks of >= HEAD_CHUNK_MIN_ROWS rows
# (tools/head_bench.py, B200, 8192 tokens x V 32000: 1 chunk 4.90 ms, 2 chunks 5.85 ms, 4
# chunks 7.07 ms -- a K=2048 wgrad is epilogue-bound), so chunking only bounds the memory of
# long-context microbatches (Llama-2-13B at 32K: 2 GB of logits per sequence)
HEAD_CHUNK_BYTES = 1 << 30
HEAD_CHUNK_MIN_ROWS = 8192


def _head_chunks(T: int, v_local: int, elt: int):
    """Token ranges (multiples of 128 rows) whose [rows, V/tp] logits stay within
    HEAD_CHUNK_BYTES, never shorter than HEAD_CHUNK_MIN_ROWS."""
    n = max(1, -(-T * v_local * elt // HEAD_CHUNK_BYTES))
    step = max(-(-T // n), min(T, HEAD_CHUNK_MIN_ROWS))
    step = -(-step // 128) * 128
    return [(a, min(T, a + step)) for a in range(0, T, step)]


class Head:
    """Final norm + vocab-parallel LM head + fused cross-entropy (last layer's layout)."""

    def __init__(self, cfg, strategy, topo, *, dtype, grad_dtype, device):
        self.cfg, self.s, self.dtype = cfg, strategy, dtype
        self.tpg, self.dpg = topo.tp(strategy.tp), topo.dp(strategy.tp)
        self.tp, self.tpr = strategy.tp, self.tpg.index
        self.vl = cfg.vocab // self.tp
        entries = [("final_norm.weight", (cfg.hidden,))]
        if cfg.arch == "gpt":
            entries.append(("final_norm.bias", (cfg.hidden,)))
        entries.append(("lm_head.weight", (self.vl, cfg.hidden)))
        # follows the last layer's ZeRO stage (charged to it by fold_embedding_head)
        self.store = ParamStore(entries, dtype=dtype, grad_dtype=grad_dtype, device=device,
                                dp=self.dpg, zero=strategy.zero_stage,
                                small_names=("final_norm.weight", "final_norm.bias"))
        self.tp_partial = ["final_norm.weight", "final_norm.bias"] if strategy.sp else []

    def forward_backward(self, x, labels, grad_scale):
        """x [T_in, h], labels [T_rep] -> (sum of token losses (fp32 tensor), dx)."""
        cfg = self.cfg
        w = self.store.views(self.store.materialize())
        gflat = self.store.grad_target()
        gw = self.store.views(gflat)
        sg = self.store.small_grads()
        gpt = cfg.arch == "gpt"
        if gpt:
            n, mean, rstd = K.layernorm_fwd(x, w["final_norm.weight"], w["final_norm.bias"],
                                            cfg.norm_eps)
        else:
            n, rstd = K.rmsnorm_fwd(x, w["final_norm.weight"], cfg.norm_eps)
            mean = None
        sp = self.s.sp and self.tp > 1
        nf = comm.all_gather(n, self.tpg) if sp else n
        T = nf.shape[0]
        stats = torch.empty(T, 3, dtype=torch.float32, device=x.device)
        loss = torch.empty(T, dtype=torch.float32, device=x.device)
        dnf = torch.empty_like(nf)
        lo = self.tpr * self.vl
        # token chunks bound the [tokens, V/tp] logits working set (HEAD_CHUNK_BYTES): each
        # chunk runs GEMM -> cross-entropy (dlogits in place) -> dgrad -> wgrad accumulate
        for a, b in _head_chunks(T, self.vl, nf.element_size()):
            logits = _linear(nf[a:b], w["lm_head.weight"])
            st, ls, lab = stats[a:b], loss[a:b], labels[a:b]
            if self.tp == 1:
                K.xent(logits, lab, st, 3, loss=ls, dlogits=logits, vocab_lo=lo,
                       grad_scale=grad_scale)
            else:
                import torch.distributed as dist
                K.xent(logits, lab, st, 0, vocab_lo=lo)
                mx = st[:, 0].contiguous()
                comm.all_reduce(mx, self.tpg, op=dist.ReduceOp.MAX)
                st[:, 0] = mx
                K.xent(logits, lab, st, 1, vocab_lo=lo)
                part = st[:, 1:3].contiguous()
                comm.all_reduce(part, self.tpg)
                st[:, 1:3] = part
                K.xent(logits, lab, st, 2, loss=ls, dlogits=logits, vocab_lo=lo,
                       grad_scale=grad_scale)
            _dgrad(logits, w["lm_head.weight"], out=dnf[a:b])
            _wgrad(logits, nf[a:b], gw["lm_head.weight"])
            del logits
        if self.tp > 1:
            dn = comm.reduce_scatter(dnf, self.tpg) if sp else comm.all_reduce(dnf, self.tpg)
        else:
            dn = dnf
        if gpt:
            dx = K.layernorm_bwd(x, w["final_norm.weight"], mean, rstd, dn,
                                 sg["final_norm.weight"], sg["final_norm.bias"])
        else:
            dx = K.rmsnorm_bwd(x, w["final_norm.weight"], rstd, dn, sg["final_norm.weight"])
        self.store.release()
        self.store.finish_microbatch(gflat, self.tp_partial, self.tpg)
        return loss.sum(), dx
