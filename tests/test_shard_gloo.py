"""Multi-shard host logic on the CPU (no GPU): the library's sharding rules
(ankh_shard_*_v1, csrc/shard.cpp) must count every P2P pair and every M2L
instance exactly once across shards.  The world-size-2 test runs two
processes over torch.distributed/gloo: each evaluates the oracle energy of
exactly the work the library assigns to its shard, the partial energies are
all-reduced, and the sum must equal the single-shard oracle energy."""
import ctypes
import os

import numpy as np
import pytest

import ankh_oracle as O
import paper_2212_08284_b200 as ankh
from paper_2212_08284_b200 import inputs


def lib():
    return ankh.lib()


def leaf_owner(depth, world):
    n = 8 ** depth
    return np.array([lib().ankh_shard_cell_owner_v1(depth, c, depth, world) for c in range(n)])


def m2l_instances(depth, periodic, rank, world):
    cnt = ctypes.c_size_t(0)
    assert lib().ankh_shard_m2l_instances_v1(depth, int(periodic), rank, world, None, None, None,
                                              None, 0, ctypes.byref(cnt)) == 0
    n = cnt.value
    lv = np.zeros(max(n, 1), np.uint32)
    t = np.zeros(max(n, 1), np.uint32)
    s = np.zeros(max(n, 1), np.uint32)
    off = np.zeros(max(3 * n, 1), np.int32)
    P32 = ctypes.POINTER(ctypes.c_uint32)
    assert lib().ankh_shard_m2l_instances_v1(
        depth, int(periodic), rank, world, lv.ctypes.data_as(P32), t.ctypes.data_as(P32),
        s.ctypes.data_as(P32), off.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n,
        ctypes.byref(cnt)) == 0
    return lv[:n], t[:n], s[:n], off[:3 * n].reshape(n, 3)


def morton(i, j, k):
    m = 0
    for b in range(10):
        m |= ((i >> b) & 1) << (3 * b + 2) | ((j >> b) & 1) << (3 * b + 1) | ((k >> b) & 1) << (3 * b)
    return m


@pytest.mark.parametrize("depth,world", [(1, 2), (2, 2), (2, 3), (2, 8), (3, 4), (3, 7)])
def test_leaf_ownership_partition(depth, world):
    owner = leaf_owner(depth, world)
    n = 1 << depth
    for r in range(world):
        b, e = ctypes.c_int64(), ctypes.c_int64()
        assert lib().ankh_shard_leaf_range_v1(depth, r, world, ctypes.byref(b), ctypes.byref(e)) == 0
        for c in range(8 ** depth):
            i, j, k = c // (n * n), (c // n) % n, c % n
            m = morton(i, j, k)
            assert (b.value <= m < e.value) == (owner[c] == r)


@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 24000, 1029000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_src_slices_partition(n, world):
    """The moment slices of collective-attached shards cover [0, n) exactly
    once, in rank order, at 256-particle block boundaries."""
    i0, i1 = ctypes.c_size_t(), ctypes.c_size_t()
    prev = 0
    for r in range(world):
        assert lib().ankh_shard_src_slice_v1(n, r, world, ctypes.byref(i0), ctypes.byref(i1)) == 0
        assert i0.value == prev and i1.value >= i0.value
        assert i0.value % 256 == 0
        prev = i1.value
    assert prev == n


@pytest.mark.parametrize("depth,world,want", [(3, 2, 1), (3, 8, 1), (5, 4, 1), (3, 16, 2), (5, 64, 2),
                                              (3, 512, 3)])
def test_exchange_level(depth, world, want):
    """Own-subtree M2M reaches down to the lowest level that splits evenly."""
    l0 = lib().ankh_shard_exchange_level_v1(depth, world)
    assert l0 == want and (8 ** l0) % world == 0
    assert l0 == 1 or (8 ** (l0 - 1)) % world != 0


@pytest.mark.parametrize("depth,periodic,world", [(2, True, 2), (2, False, 3), (3, True, 4), (3, False, 8)])
def test_m2l_instances_partition(depth, periodic, world):
    full = m2l_instances(depth, periodic, -1, 1)
    key = lambda lv, t, s, off: set(zip(lv.tolist(), t.tolist(), s.tolist(), map(tuple, off.tolist())))
    full_set = key(*full)
    assert len(full_set) == len(full[0])
    union = set()
    total = 0
    for r in range(world):
        part = m2l_instances(depth, periodic, r, world)
        ps = key(*part)
        assert not (ps & union)
        union |= ps
        total += len(part[0])
    assert union == full_set and total == len(full_set)
    # the full set is the reference's canonical instance set (fmm.cpp:244-253)
    want = set()
    for level in range(1, depth + 1):
        t, s, img = O.lambda_list(level, periodic)
        canon = (t < s) | ((t == s) & O.image_lex_positive(img))
        offs = O.instance_offset(level, t[canon], s[canon], img[canon])
        want |= set(zip([level] * int(canon.sum()), t[canon].tolist(), s[canon].tolist(),
                        map(tuple, offs.tolist())))
    assert want == full_set


def half_shell_pairs(buckets, depth, periodic, owned_leaves, r_b):
    """The GPU's P2P rule (csrc/k_p2p.cu): own triangle + 13 lex-positive neighbours."""
    n = 1 << depth
    ix, iy, sh = [], [], []
    dirs = [(dx, dy, dz) for dx in (0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
            if dx > 0 or (dx == 0 and (dy > 0 or (dy == 0 and dz > 0)))]
    assert len(dirs) == 13
    for a in owned_leaves:
        ba = buckets[a]
        if len(ba) == 0:
            continue
        x, y = np.triu_indices(len(ba), k=1)
        ix.append(ba[x]); iy.append(ba[y]); sh.append(np.zeros((len(x), 3)))
        ai = (a // (n * n), (a // n) % n, a % n)
        for d in dirs:
            ext = [ai[k] + d[k] for k in range(3)]
            if not periodic and any(e < 0 or e >= n for e in ext):
                continue
            img = [e // n for e in ext]  # floor division == split_extended for |d| <= 1
            inb = [e - n * g for e, g in zip(ext, img)]
            b = (inb[0] * n + inb[1]) * n + inb[2]
            bb = buckets[b]
            if len(bb) == 0:
                continue
            ix.append(np.repeat(ba, len(bb))); iy.append(np.tile(bb, len(ba)))
            sh.append(np.broadcast_to(2.0 * r_b * np.array(img, float), (len(ba) * len(bb), 3)))
    if not ix:
        return None
    return np.concatenate(ix), np.concatenate(iy), np.concatenate(sh)


def shard_energy(rank, world, pos, src, r_b, depth, L, periodic, xi=0.01, p=15):
    buckets = O.build_tree(pos, r_b, depth)
    owner = leaf_owner(depth, world)
    owned = np.nonzero(owner == rank)[0]
    e_near = 0.0
    pr = half_shell_pairs(buckets, depth, periodic, owned, r_b)
    if pr is not None:
        ix, iy, sh = pr
        e_near = float(O.pair_interaction(pos[ix], src[ix], pos[iy] + sh, src[iy], xi).sum())
    exps = O.upward_pass(O.leaf_expansions(pos, src, r_b, buckets, depth, L), depth, L)
    lv, t, s, off = m2l_instances(depth, periodic, rank, world)
    e_far = 0.0
    cache = {}
    for i in range(len(lv)):
        key = (int(lv[i]), tuple(off[i]))
        if key not in cache:
            rad = r_b / (1 << key[0])
            kk = O.offset_key(key[1])
            cache[key] = O.compress_m2l(O.m2l_dense(L, rad, key[1], xi), 1e-7, O.m2l_seed(key[0], kk))
        lm, rm = cache[key]
        e_far += float((lm @ exps[key[0]][t[i]]) @ (rm @ exps[key[0]][s[i]]))
    e_self = O.self_energy(src, xi) if rank == 0 else 0.0
    e_per = O.periodic_far_energy(exps[0][0], r_b, L, xi, p) if (rank == 0 and periodic) else 0.0
    return np.array([e_self, e_near, e_far, e_per])


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    pos, src = inputs.random_system(700, 5.0, seed=3, multipoles=True)
    part = torch.from_numpy(shard_energy(rank, world, pos, src, 5.0, 2, 3, True))
    dist.all_reduce(part)
    if rank == 0:
        np.save(out_path, part.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_shards_gloo_allreduce(tmp_path):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "e.npy")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    pos, src = inputs.random_system(700, 5.0, seed=3, multipoles=True)
    want = O.fmm_energy(pos, src, 5.0, order_cheb=3, order_equi=3, depth=2, p=15)
    comps = abs(want["e_near"]) + abs(want["e_far"]) + abs(want["e_self"])
    assert abs(got[1] - want["e_near"]) <= 1e-12 * comps
    assert abs(got[2] - want["e_far"]) <= 1e-12 * comps
    assert abs(got.sum() - want["e_total"]) <= 1e-11 * comps


def halo_cells(level, depth, periodic, src, dst, world):
    cnt = ctypes.c_size_t(0)
    assert lib().ankh_shard_halo_cells_v1(level, depth, int(periodic), src, dst, world, None, 0,
                                           ctypes.byref(cnt)) == 0
    out = np.zeros(max(cnt.value, 1), np.uint32)
    assert lib().ankh_shard_halo_cells_v1(level, depth, int(periodic), src, dst, world,
                                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                           cnt.value, ctypes.byref(cnt)) == 0
    return set(int(v) for v in out[:cnt.value])


@pytest.mark.parametrize("depth,world,periodic", [(3, 2, True), (3, 8, True), (4, 8, True),
                                                  (4, 4, False), (4, 64, True), (3, 8, False)])
def test_halo_covers_every_m2l_read(depth, world, periodic):
    """Every cell a shard's M2L instances read at a halo level is either its
    own or in the halo list its owner sends it, and halo lists
    hold only the sender's own cells."""
    lh = lib().ankh_shard_exchange_level_v1(depth, world) + 1
    for r in range(world):
        lv, t, s, off = m2l_instances(depth, periodic, r, world)
        for level in range(lh, depth + 1):
            n = 1 << level
            cells = 8 ** level
            own = lambda m, q: cells * q // world <= m < cells * (q + 1) // world
            sel = lv == level
            recv = {q: halo_cells(level, depth, periodic, q, r, world) for q in range(world) if q != r}
            for q, hs in recv.items():
                assert all(own(m, q) for m in hs)
            for c in np.concatenate([t[sel], s[sel]]):
                c = int(c)
                m = morton(c // (n * n), (c // n) % n, c % n)
                if own(m, r):
                    continue
                q = m * world // cells
                assert m in recv[q], (level, r, q, m)


def test_halo_exchange_bytes_config4():
    """§8e: at config 4 (depth 6, L = 5) on 8 GPUs a shard receives <= 30 MB
    per evaluation (20.0 MB; the whole-level all-gather received 235 MB); at
    config 3 (depth 5) 5.8 MB instead of 29.4 MB."""
    def bytes_(depth, rank, halo):
        rv, sd = ctypes.c_size_t(), ctypes.c_size_t()
        assert lib().ankh_shard_exchange_bytes_v1(depth, 1, 5, rank, 8, int(halo), ctypes.byref(rv),
                                                  ctypes.byref(sd)) == 0
        return rv.value, sd.value
    for r in range(8):
        h4, _ = bytes_(6, r, True)
        a4, _ = bytes_(6, r, False)
        assert h4 <= 30e6, h4
        assert a4 > 200e6
        h3, _ = bytes_(5, r, True)
        a3, _ = bytes_(5, r, False)
        assert h3 < 0.5 * a3, (h3, a3)
