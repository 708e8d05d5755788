"""oracle/model_ref.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

CPU fp32 restatement of the policy / PRM forward the B200 path runs for every
decode row and every scored thought (paper_2605_10195_b200/csrc/model_*.{cu,cpp}).

Parity status: **unpinned against the reference** — the reference simulator has
no model at all (decode is a virtual clock and the reward a
hash oracle), so this restatement is the only oracle for model arithmetic. It is
independent of the device's incremental tree-KV mechanics: it recomputes a row
by a full causal forward over the row's root -> node token sequence, rebuilt from
the event log (node records) and the query seeds.

Quantisation points mirror the device exactly (bf16 weights; bf16 RMSNorm
outputs, K/V cache, attention output and SwiGLU output; fp32 everything else),
so the remaining differences are fp32 accumulation order and a few ulps of
sin/cos/exp — see tests/test_model_gpu.py for the stated tolerances.
"""
from __future__ import annotations

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
SALT_TOK = 0x746F6B5F69647300


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def extend_hash(h: int, slot: int) -> int:
    """rng.hpp:30-33."""
    v = (slot + 1) & 0xFFFFFFFFFFFFFFFF
    return splitmix64(h ^ ((v + 0x9E3779B97F4A7C15 + (h << 6) + (h >> 2)) & 0xFFFFFFFFFFFFFFFF))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, like __float2bfloat16_rn."""
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32)


def init_tensor(n: int, seed: int, tensor_id: int, scale: float) -> np.ndarray:
    """init_weights_kernel: uniform counter-hash weights, bf16-rounded."""
    i = np.arange(n, dtype=np.uint64)
    h = _splitmix64_np((np.uint64(tensor_id) << np.uint64(40)) ^ i ^ np.uint64(seed))
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(5.9604644775390625e-08)
    v = (u * np.float32(2.0) - np.float32(1.0)) * np.float32(scale)
    return bf16_round(v)


def token_id(node_hash: int, pos: int, V: int) -> int:
    h = splitmix64(node_hash ^ (((pos + 1) * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF) ^ SALT_TOK)
    return h % V


SHAPES = {
    # d, L, H, KVH, dh, F, V, rope_theta, eps   (model_host.cpp: shape_by_name)
    "small_policy": (256, 2, 4, 2, 64, 768, 512, 10000.0, 1e-5),
    "small_prm": (128, 2, 2, 2, 64, 384, 512, 10000.0, 1e-5),
    "mid_policy": (1024, 8, 8, 8, 128, 2816, 32000, 10000.0, 1e-5),
    "mid_prm": (512, 4, 4, 4, 128, 1408, 32000, 10000.0, 1e-5),
}

PRM_SEED_XOR = 0x50524D00


class Model:
    def __init__(self, shape: str, seed: int, prm: bool):
        d, L, H, KVH, dh, F, V, theta, eps = SHAPES[shape]
        self.d, self.L, self.H, self.KVH, self.dh, self.F, self.V = d, L, H, KVH, dh, F, V
        self.theta, self.eps, self.prm = theta, eps, prm
        std = np.float32(0.02 * 1.7320508)
        self.embed = init_tensor(V * d, seed, 1, np.float32(1.7320508)).reshape(V, d)
        self.layers = []
        for l in range(L):
            nq = (H + 2 * KVH) * dh
            self.layers.append(dict(
                wqkv=init_tensor(nq * d, seed, 100 + 8 * l + 0, std).reshape(nq, d),
                wo=init_tensor(d * H * dh, seed, 100 + 8 * l + 1, std).reshape(d, H * dh),
                wgu=init_tensor(2 * F * d, seed, 100 + 8 * l + 2, std).reshape(2 * F, d),
                wd=init_tensor(d * F, seed, 100 + 8 * l + 3, std).reshape(d, F),
            ))
        if prm:
            self.vhead = init_tensor(d, seed, 3, std)
        else:
            self.lm = init_tensor(V * d, seed, 2, std).reshape(V, d)
        self.inv_freq = (1.0 / np.power(float(theta), (2.0 * np.arange(dh // 2)) / dh)).astype(np.float32)

    def _rms(self, x):
        ms = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True, dtype=np.float32)
        return bf16_round(x * (np.float32(1.0) / np.sqrt(ms + np.float32(self.eps))))

    def _rope(self, x, pos):
        half = self.dh // 2
        ang = pos[:, None].astype(np.float32) * self.inv_freq[None, :]
        c, s = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
        a, b = x[..., :half], x[..., half:]
        return np.concatenate([a * c[:, None, :] - b * s[:, None, :], a * s[:, None, :] + b * c[:, None, :]], axis=-1)

    def forward(self, tokens: np.ndarray) -> np.ndarray:
        """Full causal forward; returns the final-normed bf16 hidden states [T, d]."""
        T = len(tokens)
        H, KVH, dh, G = self.H, self.KVH, self.dh, self.H // self.KVH
        pos = np.arange(T)
        X = self.embed[tokens].astype(np.float32)
        mask = np.triu(np.ones((T, T), dtype=bool), 1)
        for lw in self.layers:
            xn = self._rms(X)
            qkv = xn @ lw["wqkv"].T
            q = qkv[:, : H * dh].reshape(T, H, dh)
            k = qkv[:, H * dh: (H + KVH) * dh].reshape(T, KVH, dh)
            v = qkv[:, (H + KVH) * dh:].reshape(T, KVH, dh)
            q = self._rope(q, pos) * np.float32(1.0 / np.sqrt(dh))
            k = bf16_round(self._rope(k, pos))
            v = bf16_round(v)
            o = np.empty((T, H, dh), dtype=np.float32)
            for h in range(H):
                kh = h // G
                s = (q[:, h, :] @ k[:, kh, :].T).astype(np.float32)
                s[mask] = -np.inf
                s = s - s.max(axis=1, keepdims=True)
                p = np.exp(s).astype(np.float32)
                p /= p.sum(axis=1, keepdims=True)
                o[:, h, :] = p @ v[:, kh, :]
            X = X + bf16_round(o.reshape(T, H * dh)) @ lw["wo"].T
            xn = self._rms(X)
            gu = xn @ lw["wgu"].T
            g, u = gu[:, : self.F], gu[:, self.F:]
            a = bf16_round(g / (np.float32(1.0) + np.exp(-g)) * u)
            X = X + a @ lw["wd"].T
        return self._rms(X)

    def logits_stats(self, tokens: np.ndarray):
        h = self.forward(tokens)[-1]
        z = (h @ self.lm.T).astype(np.float64)
        m = z.max()
        return int(np.argmax(z)), float(m + np.log(np.exp(z - m).sum())), float(z.sum()), z

    def prm_score(self, tokens: np.ndarray) -> float:
        h = self.forward(tokens)[-1]
        t = float(np.dot(h.astype(np.float64), self.vhead.astype(np.float64)))
        return 1.0 / (1.0 + np.exp(-t))


class TreeFromLog:
    """Rebuilds node parents / token counts / path hashes from an event log."""

    def __init__(self, lines, prompt_tokens: int):
        import json
        self.prompt = prompt_tokens
        self.seed = {}
        self.nodes = {}  # (q, node) -> (parent, slot, tokens)
        for ln in lines:
            e = json.loads(ln)
            if e["ev"] == "admit":
                self.seed[e["q"]] = e["seed"]
            elif e["ev"] == "node":
                self.nodes[(e["q"], e["node"])] = (e["parent"], e["slot"], e["tokens"])
        self._hash = {}

    def path_hash(self, q: int, node: int) -> int:
        key = (q, node)
        if key in self._hash:
            return self._hash[key]
        if node == 0:
            h = splitmix64(self.seed[q])
        else:
            parent, slot, _ = self.nodes[key]
            h = extend_hash(self.path_hash(q, parent), slot)
        self._hash[key] = h
        return h

    def chain(self, q: int, node: int):
        out = []
        while node != 0:
            out.append(node)
            node = self.nodes[(q, node)][0]
        return out[::-1]

    def sequence(self, q: int, node: int, upto: int, V: int) -> np.ndarray:
        """Token ids of prompt + every ancestor thought + node tokens [0, upto]."""
        toks = [token_id(self.path_hash(q, 0), j, V) for j in range(self.prompt)]
        for a in self.chain(q, node)[:-1] if node != 0 else []:
            n = self.nodes[(q, a)][2]
            ha = self.path_hash(q, a)
            toks += [token_id(ha, j, V) for j in range(n)]
        if node != 0:
            hn = self.path_hash(q, node)
            toks += [token_id(hn, j, V) for j in range(upto + 1)]
        return np.asarray(toks, dtype=np.int64)
