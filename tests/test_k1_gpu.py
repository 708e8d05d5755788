"""K1 tree decode attention vs a plain PyTorch fp32 reference of the same op.

The kernel (`spex_k_tree_attn`, model_kernels.cu) is called directly through
the product library on random paged tree KV pools: each row attends over a
list of KV segments (its ancestors' thoughts root-first, then its own prefix),
segments shared between rows as siblings share ancestors. The reference
gathers each row's K/V in fp32 and computes softmax(q.K^T).V.

Tolerance (stated): the kernels take q and p in bf16 (the tensor-core tile
kernel's mma operands, the decode kernel's FHFMA operands) and write O in bf16,
so |O - O_ref| <= 2e-2 (1 + |O_ref|) elementwise and mean |O - O_ref| <= 2e-3.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROW = np.dtype([("q", "<i4"), ("node", "<u4"), ("pos", "<i4"), ("abs_pos", "<i4"), ("slot", "<i8"),
                ("seg_off", "<i4"), ("nseg", "<i4"), ("token", "<i4"), ("pad", "<i4")])
SEG = np.dtype([("base", "<i8"), ("len", "<i4"), ("own0", "<i4")])
MAX_SEG = 40
N_QUERIES = 5  # rows are spread over a few queries


def _lib():
    import paper_2605_10195_b200 as spex
    from paper_2605_10195_b200 import _lib as L
    if not spex.device_ok():
        pytest.fail("no sm_100 device: the B200 path has no fallback")
    lib = L.lib()
    f = lib.spex_k_tree_attn
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int,
                  ctypes.c_void_p]
    return f


def _make_tree_rows(rng, M, slots, max_depth):
    """Random tree: nodes own contiguous slot ranges; each row is a path
    root->...->node with the last segment a partial own prefix."""
    n_nodes = max(8, M // 2)
    lens = rng.integers(8, 200, size=n_nodes)
    bases = np.concatenate([[0], np.cumsum(lens)[:-1]])
    assert bases[-1] + lens[-1] <= slots
    parent = np.full(n_nodes, -1)
    for i in range(1, n_nodes):
        parent[i] = rng.integers(0, i) if rng.random() < 0.9 else -1
    rows = np.zeros(M, ROW)
    segs = np.zeros(M * MAX_SEG, SEG)
    paths = []
    for r in range(M):
        node = int(rng.integers(0, n_nodes))
        chain = []
        c = parent[node]
        while c >= 0 and len(chain) < max_depth:
            chain.append(c)
            c = parent[c]
        chain = chain[::-1]
        own = int(rng.integers(1, lens[node] + 1))
        sl = [(int(bases[a]), int(lens[a])) for a in chain] + [(int(bases[node]), own)]
        for k, (b, n) in enumerate(sl):
            segs[r * MAX_SEG + k] = (b, n, -1 if k < len(sl) - 1 else 0)
        rows[r] = (int(rng.integers(0, N_QUERIES)), node, own - 1, 0, bases[node] + own - 1, r * MAX_SEG,
                   len(sl), 0, 0)
        paths.append(sl)
    return rows, segs, paths


@pytest.mark.parametrize("impl", ["row", "bulk", "wmma"])
@pytest.mark.parametrize("H,KVH,dh,M", [(8, 8, 128, 300), (32, 8, 128, 97), (12, 2, 128, 80), (4, 2, 64, 150), (16, 4, 64, 64)])
def test_k1_decode_matches_torch_fp32(H, KVH, dh, M, impl):
    """impl "row": one warp per (row, kv head), register pipeline (spex_k_tree_attn);
    "bulk": the bulk-copy pipeline (G = 1), launched twice to exercise its
    self-resetting work counter; "wmma": the per-warp TMA + tensor-core
    pipeline (GQA groups)."""
    import torch
    f = _lib()
    rng = np.random.default_rng(H * 1000 + dh + M)
    slots = 200 * max(8, M // 2) + 64
    rows, segs, paths = _make_tree_rows(rng, M, slots, max_depth=12)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(M)
    K = torch.randn(KVH, slots, dh, generator=g).to(torch.bfloat16).to(dev)
    V = torch.randn(KVH, slots, dh, generator=g).to(torch.bfloat16).to(dev)
    Q = (torch.randn(M, H, dh, generator=g) * 2.0 / dh ** 0.5).to(dev)  # pre-scaled like rope_kv_kernel
    O = torch.zeros(M, H, dh, dtype=torch.bfloat16, device=dev)
    rows_d = torch.from_numpy(rows.view(np.uint8).copy()).to(dev)
    segs_d = torch.from_numpy(segs.view(np.uint8).copy()).to(dev)
    st = torch.cuda.current_stream(dev)
    if impl == "row":
        rc = f(rows_d.data_ptr(), segs_d.data_ptr(), Q.data_ptr(), H, KVH, dh, K.data_ptr(), V.data_ptr(), slots,
               O.data_ptr(), M, st.cuda_stream)
        assert rc == 0
    elif impl == "wmma":
        if dh != 128:
            pytest.skip("per-warp TMA decode kernel is dh=128")
        from paper_2605_10195_b200 import _lib as L
        lib = L.lib()
        lib.spex_tmap_kv16.restype = ctypes.c_int
        lib.spex_tmap_kv16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                       ctypes.c_int]
        fw = lib.spex_k_tree_attn_wmma
        fw.restype = ctypes.c_int
        fw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int,
                       ctypes.c_void_p, ctypes.c_void_p]
        # the pools' K|V pair as one map: V must sit above K (one allocation, as the model's pools)
        KV = torch.stack([K, V])
        K, V = KV[0], KV[1]
        km = ctypes.create_string_buffer(256)
        kp = (ctypes.addressof(km) + 63) & ~63
        assert lib.spex_tmap_kv16(kp, K.data_ptr(), V.data_ptr(), KVH * slots, dh) == 0
        assert lib.spex_tmap_kv16(kp, V.data_ptr(), K.data_ptr(), KVH * slots, dh) != 0  # V below K: refused
        assert lib.spex_tmap_kv16(kp, K.data_ptr(), V.data_ptr(), KVH * slots, dh) == 0
        ctr = torch.zeros(1, dtype=torch.int32, device=dev)
        rc = fw(kp, rows_d.data_ptr(), segs_d.data_ptr(), Q.data_ptr(), H, KVH, dh, slots, O.data_ptr(), M,
                ctr.data_ptr(), st.cuda_stream)
        assert rc == 0
    elif impl == "bulk":
        if dh != 128 or H != KVH:
            pytest.skip("bulk-copy decode kernel is dh=128, G=1")
        from paper_2605_10195_b200 import _lib as L
        fb = L.lib().spex_k_tree_attn_bulk
        fb.restype = ctypes.c_int
        fb.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int,
                       ctypes.c_void_p, ctypes.c_void_p]
        ctr = torch.zeros(2, dtype=torch.int32, device=dev)  # [claims, finished warps], self-resetting
        rc = fb(rows_d.data_ptr(), segs_d.data_ptr(), Q.data_ptr(), H, KVH, dh, K.data_ptr(), V.data_ptr(), slots,
                O.data_ptr(), M, ctr.data_ptr(), st.cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        assert ctr.tolist() == [0, 0]  # re-zeroed by the last warp
        O.zero_()
        rc = fb(rows_d.data_ptr(), segs_d.data_ptr(), Q.data_ptr(), H, KVH, dh, K.data_ptr(), V.data_ptr(), slots,
                O.data_ptr(), M, ctr.data_ptr(), st.cuda_stream)  # second launch on the reset counter
        assert rc == 0
    torch.cuda.synchronize()
    Kf, Vf = K.float(), V.float()
    G = H // KVH
    worst, tot, cnt = 0.0, 0.0, 0
    for r in range(M):
        idx = torch.cat([torch.arange(b, b + n) for b, n in paths[r]]).to(dev)
        for h in range(H):
            kh = h // G
            s = Kf[kh, idx] @ Q[r, h]
            p = torch.softmax(s, dim=0)
            ref = p @ Vf[kh, idx]
            d = (O[r, h].float() - ref).abs()
            worst = max(worst, (d / (1.0 + ref.abs())).max().item())
            tot += d.sum().item()
            cnt += d.numel()
    assert worst <= 2e-2, worst
    assert tot / cnt <= 2e-3, tot / cnt


TILE = np.dtype([("row0", "<i4"), ("nrows", "<i4")])


@pytest.mark.parametrize("H,KVH", [(8, 8), (16, 8), (32, 8), (12, 2)])
def test_k1_tile_mma_matches_torch_fp32(H, KVH):
    """PRM / prompt rows: 16 consecutive positions of one thought share one pass
    over their context (TMA-staged 64-token chunks, mma.sync), the own segment
    causally masked per row; GQA group sizes 1, 2, 4 and 6 (12/2, the 1.5B PRM)."""
    import torch
    import paper_2605_10195_b200 as spex
    from paper_2605_10195_b200 import _lib as L
    if not spex.device_ok():
        pytest.fail("no sm_100 device")
    lib = L.lib()
    lib.spex_tmap_kv.restype = ctypes.c_int
    lib.spex_tmap_kv.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int]
    f = lib.spex_k_tree_attn_tiles_mma
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p,
                  ctypes.c_void_p]
    dh = 128
    rng = np.random.default_rng(H + KVH)
    n_nodes = 24
    lens = rng.integers(8, 150, size=n_nodes)
    bases = np.concatenate([[0], np.cumsum(lens)[:-1]])
    alt0 = int(bases[-1] + lens[-1]) + 64  # second run of split thoughts (elsewhere in the pool)
    slots = alt0 + int(lens.sum()) + 64
    parent = np.full(n_nodes, -1)
    for i in range(1, n_nodes):
        parent[i] = rng.integers(0, i)
    # The product's PRM rows: one segment list per thought (ancestor runs, then
    # the thought's own runs tagged with their first position, own0), shared by
    # all its rows; the kernel clips the own runs at each tile's last row.
    # Every other thought's own tokens are split into two physical runs at a
    # page boundary, like a thought whose pages came from the free ring.
    rows, seg_lists, tiles, ctx = [], [], [], []
    for ti, node in enumerate(rng.choice(n_nodes, size=6, replace=False)):
        chain, c = [], parent[node]
        while c >= 0:
            chain.append(c)
            c = parent[c]
        anc = [(int(bases[a]), int(lens[a]), -1) for a in chain[::-1]]
        n = int(lens[node])
        split = 16 * (1 + int(rng.integers(0, max(1, (n - 1) // 16)))) if ti % 2 == 0 and n > 16 else n
        own = [(int(bases[node]), split, 0)] + ([(alt0 + int(bases[node]), n - split, split)] if split < n else [])
        sl = anc + own
        off = len(seg_lists)
        seg_lists.extend(sl)
        anc_idx = [b + t for (b, ln, _) in anc for t in range(ln)]
        own_idx = [int(bases[node]) + t if t < split else alt0 + int(bases[node]) + (t - split) for t in range(n)]
        for j0 in range(0, n, 16):
            tiles.append((len(rows), min(16, n - j0)))
            for j in range(j0, min(n, j0 + 16)):
                rows.append((0, node, j, 0, own_idx[j], off, len(sl), 0, 0))
                ctx.append(anc_idx + own_idx[: j + 1])
    M = len(rows)
    rows_np = np.array(rows, ROW)
    segs_np = np.zeros(max(len(seg_lists), 1), SEG)
    for k, (b, ln, o) in enumerate(seg_lists):
        segs_np[k] = (b, ln, o)
    tiles_np = np.array(tiles, TILE)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(H * 7 + KVH)
    K = torch.randn(KVH, slots, dh, generator=g).to(torch.bfloat16).to(dev)
    V = torch.randn(KVH, slots, dh, generator=g).to(torch.bfloat16).to(dev)
    Q = (torch.randn(M, H, dh, generator=g) * 2.0 / dh ** 0.5).to(dev)
    O = torch.zeros(M, H, dh, dtype=torch.bfloat16, device=dev)
    bufs = [torch.from_numpy(a.view(np.uint8).copy()).to(dev) for a in (rows_np, segs_np, tiles_np)]
    KV = torch.stack([K, V])  # the pools' K|V pair as one map: V above K, as the model allocates them
    K, V = KV[0], KV[1]
    km = ctypes.create_string_buffer(256)
    kp = (ctypes.addressof(km) + 63) & ~63
    assert lib.spex_tmap_kv(kp, K.data_ptr(), V.data_ptr(), KVH * slots, dh) == 0
    st = torch.cuda.current_stream(dev)
    rc = f(kp, bufs[2].data_ptr(), len(tiles), bufs[0].data_ptr(), bufs[1].data_ptr(), Q.data_ptr(), H, KVH, dh,
           slots, O.data_ptr(), st.cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    Kf, Vf = K.float(), V.float()
    G = H // KVH
    worst = 0.0
    for r in range(M):
        idx = torch.as_tensor(ctx[r], device=dev)
        for h in range(H):
            kh = h // G
            p = torch.softmax(Kf[kh, idx] @ Q[r, h], dim=0)
            ref = p @ Vf[kh, idx]
            worst = max(worst, ((O[r, h].float() - ref).abs() / (1.0 + ref.abs())).max().item())
    assert worst <= 2e-2, worst
