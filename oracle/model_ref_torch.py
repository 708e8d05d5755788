"""oracle/model_ref_torch.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

The fp32 restatement of oracle/model_ref.py (numpy) written with torch ops so it
can check the named model shapes (Llama-3-8B-shaped policy, 1.5B-shaped PRM)
that numpy on the host cannot run in test time. Same arithmetic, same
quantisation points (bf16 weights; bf16 RMSNorm outputs, K/V, attention output
and SwiGLU output; fp32 everything else), same counter-hash weights, same
teacher-forced token ids; full causal forward over a row's root -> node token
sequence, independent of the device's tree-KV mechanics. Matmuls run in true
fp32 (TF32 disabled).

Pinned to oracle/model_ref.py on the small and mid shapes by
tests/test_model_oracle_cpu.py. Parity against the reference itself is
unpinned: the reference has no model.
"""
from __future__ import annotations

import math

import torch

from oracle import model_ref

SHAPES = dict(model_ref.SHAPES)
SHAPES.update({
    # d, L, H, KVH, dh, F, V, rope_theta, eps   (model_host.cpp: shape_by_name)
    "llama3_8b": (4096, 32, 32, 8, 128, 14336, 128256, 500000.0, 1e-5),
    "prm_1p5b": (1536, 28, 12, 2, 128, 8960, 128256, 1000000.0, 1e-6),
})

_M64 = (1 << 64) - 1


def _i64(c: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    c &= _M64
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """logical shift right of int64 bit patterns"""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _splitmix64(x: torch.Tensor) -> torch.Tensor:
    x = x + _i64(0x9E3779B97F4A7C15)
    x = (x ^ _lsr(x, 30)) * _i64(0xBF58476D1CE4E5B9)
    x = (x ^ _lsr(x, 27)) * _i64(0x94D049BB133111EB)
    return x ^ _lsr(x, 31)


def _bf16(x: torch.Tensor) -> torch.Tensor:
    """fp32 -> bf16 (round to nearest even) -> fp32"""
    return x.to(torch.bfloat16).to(torch.float32)


def init_tensor(n: int, seed: int, tensor_id: int, scale: float, device) -> torch.Tensor:
    """model_ref.init_tensor (init_weights_kernel) on `device`, as bf16."""
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    chunk = 1 << 26
    base = _i64((tensor_id << 40) ^ seed)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        i = torch.arange(s, e, dtype=torch.int64, device=device)
        h = _splitmix64(i ^ base)
        u = _lsr(h, 40).to(torch.float32) * 5.9604644775390625e-08
        out[s:e] = ((u * 2.0 - 1.0) * scale).to(torch.bfloat16)
    return out


class Model:
    """Weights kept as bf16 (their exact values), upcast to fp32 per matmul."""

    def __init__(self, shape: str, seed: int, prm: bool, device="cpu"):
        d, L, H, KVH, dh, F, V, theta, eps = SHAPES[shape]
        self.d, self.L, self.H, self.KVH, self.dh, self.F, self.V = d, L, H, KVH, dh, F, V
        self.theta, self.eps, self.prm, self.device = theta, eps, prm, device
        std = 0.02 * 1.7320508
        # float32 constants as numpy computes them (np.float32(0.02 * 1.7320508))
        std = float(torch.tensor(std, dtype=torch.float32))
        esc = float(torch.tensor(1.7320508, dtype=torch.float32))
        self.embed = init_tensor(V * d, seed, 1, esc, device).view(V, d)
        self.layers = []
        for l in range(L):
            nq = (H + 2 * KVH) * dh
            self.layers.append(dict(
                wqkv=init_tensor(nq * d, seed, 100 + 8 * l + 0, std, device).view(nq, d),
                wo=init_tensor(d * H * dh, seed, 100 + 8 * l + 1, std, device).view(d, H * dh),
                wgu=init_tensor(2 * F * d, seed, 100 + 8 * l + 2, std, device).view(2 * F, d),
                wd=init_tensor(d * F, seed, 100 + 8 * l + 3, std, device).view(d, F),
            ))
        if prm:
            self.vhead = init_tensor(d, seed, 3, std, device)
        else:
            self.lm = init_tensor(V * d, seed, 2, std, device).view(V, d)
        inv = 1.0 / torch.pow(torch.tensor(float(theta), dtype=torch.float64),
                              (2.0 * torch.arange(dh // 2, dtype=torch.float64)) / dh)
        self.inv_freq = inv.to(torch.float32).to(device)

    @staticmethod
    def _mm(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        return x @ w.to(torch.float32).T

    def _rms(self, x: torch.Tensor) -> torch.Tensor:
        ms = torch.mean(x * x, dim=-1, keepdim=True)
        return _bf16(x * (1.0 / torch.sqrt(ms + self.eps)))

    def _rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        half = self.dh // 2
        ang = pos[:, None].to(torch.float32) * self.inv_freq[None, :]
        c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        a, b = x[..., :half], x[..., half:]
        return torch.cat([a * c - b * s, a * s + b * c], dim=-1)

    @torch.no_grad()
    def forward(self, tokens) -> torch.Tensor:
        """Full causal forward; returns the final-normed bf16-valued hidden states [T, d] (fp32)."""
        dev = self.device
        toks = torch.as_tensor(tokens, dtype=torch.int64, device=dev)
        T = toks.numel()
        H, KVH, dh, G = self.H, self.KVH, self.dh, self.H // self.KVH
        pos = torch.arange(T, device=dev)
        X = self.embed[toks].to(torch.float32)
        mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=dev), 1)
        scale = float(torch.tensor(1.0 / math.sqrt(dh), dtype=torch.float32))
        for lw in self.layers:
            xn = self._rms(X)
            qkv = self._mm(xn, lw["wqkv"])
            q = qkv[:, : H * dh].reshape(T, H, dh)
            k = qkv[:, H * dh: (H + KVH) * dh].reshape(T, KVH, dh)
            v = qkv[:, (H + KVH) * dh:].reshape(T, KVH, dh)
            q = self._rope(q, pos) * scale
            k = _bf16(self._rope(k, pos))
            v = _bf16(v)
            kk = k.repeat_interleave(G, dim=1).permute(1, 2, 0)  # [H, dh, T]
            vv = v.repeat_interleave(G, dim=1).permute(1, 0, 2)  # [H, T, dh]
            s = torch.bmm(q.permute(1, 0, 2), kk)  # [H, T, T]
            s.masked_fill_(mask, float("-inf"))
            s = s - s.amax(dim=-1, keepdim=True)
            p = torch.exp(s)
            p = p / p.sum(dim=-1, keepdim=True)
            o = torch.bmm(p, vv).permute(1, 0, 2).reshape(T, H * dh)
            X = X + self._mm(_bf16(o), lw["wo"])
            xn = self._rms(X)
            gu = self._mm(xn, lw["wgu"])
            g, u = gu[:, : self.F], gu[:, self.F:]
            a = _bf16(g / (1.0 + torch.exp(-g)) * u)
            X = X + self._mm(a, lw["wd"])
        return self._rms(X)

    @torch.no_grad()
    def logits_stats_all(self, tokens, positions, cand=None):
        """(argmax, logsumexp, logit sum, gap) of the rows at `positions` of one
        sequence; gap[i] = z[argmax] - z[cand[i]] (the fp32 logit margin by which
        token cand[i] loses), or the top-2 gap when no candidates are given."""
        h = self.forward(tokens)[torch.as_tensor(positions, device=self.device)]
        z = self._mm(h, self.lm).to(torch.float64)
        lse = torch.logsumexp(z, dim=-1)
        top = torch.topk(z, 2, dim=-1).values
        if cand is None:
            gap = top[:, 0] - top[:, 1]
        else:
            c = torch.as_tensor(cand, device=z.device, dtype=torch.long)
            gap = top[:, 0] - z.gather(1, c[:, None])[:, 0]
        return (z.argmax(dim=-1).tolist(), lse.tolist(), z.sum(dim=-1).tolist(), gap.tolist())

    @torch.no_grad()
    def prm_score(self, tokens) -> float:
        h = self.forward(tokens)[-1]
        t = float(torch.dot(h.to(torch.float64), self.vhead.to(torch.float64)))
        return 1.0 / (1.0 + math.exp(-t))
