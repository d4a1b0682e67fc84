"""CPU, world_size 2 (gloo): the multi-GPU host orchestration (paper_2404_01159_b200.dist.ShardedRvea with
TorchComm) — exchange planning (C ABI temo_b200_shard_plan), parent all-to-all, objective / free-slot
all-gathers, packed min-allreduces, survivor table updates — driven end to end with a CPU stand-in for the
per-rank stage functions (the oracle does the arithmetic here; on the GPU it is GpuShard). The sharded run
must reproduce the single-process oracle run bit for bit: same survivor sets, same X, same F, every generation.
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

KEY_FLIP = np.uint64(0x8000000000000000)


def order_key(x):
    b = np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)
    return np.where(b >> np.uint64(63), ~b, b | KEY_FLIP)


class CpuShard:
    """Stand-in for GpuShard: same methods and buffers (CPU tensors), arithmetic by the oracle."""

    def __init__(self, cfg, rank, world, oracle):
        import ctypes as C
        from oracle.pyoracle import _p, u64
        self.C, self._p, self.u64 = C, _p, u64
        self.o, self.cfg, self.rank, self.world = oracle, cfg, rank, world
        self.n, self.d, self.m = cfg.pop, cfg.dim, cfg.obj
        H = cfg.lattice_h or oracle.lattice_density_for(self.m, self.n)
        self.v0, self.gamma = oracle.make_ref_set(self.m, H)
        self.v = self.v0.copy()
        self.r = self.v0.shape[0]
        self.n_loc = self.n // world
        self.h_loc = self.n_loc // 2
        self.pcap = max(self.n, self.r)
        self.cap_loc = self.pcap + self.n_loc
        self.send_cap = self.n
        self.adapt_every = max(1, int(np.ceil(cfg.fr * cfg.generations)))
        self.lo, self.hi = oracle.problem_bounds(cfg.problem, self.d, self.m)
        self.pool = np.zeros((self.cap_loc, self.d))
        rows0 = self.n_loc
        x, _ = oracle.random_reproduce(rows0, self.d, cfg.seed, rank * rows0 * self.d, self.lo, self.hi)
        self.pool[:rows0] = x
        self.used = np.zeros(self.cap_loc, dtype=bool)
        self.used[:rows0] = True
        self.send_buf = torch.zeros(self.send_cap, self.d, dtype=torch.float64)
        self.recv_buf = torch.zeros(self.n_loc, self.d, dtype=torch.float64)
        self.f_off_loc = torch.from_numpy(oracle.evaluate(cfg.problem, x, self.m).copy())
        self.f_gather = torch.zeros(world * self.n_loc, self.m, dtype=torch.float64)
        self.best_key = torch.zeros(self.r, dtype=torch.int64)
        self.first_row = torch.zeros(self.r, dtype=torch.int32)
        self.best_row = torch.zeros(self.r, dtype=torch.int32)
        self.free_slot = torch.from_numpy(self._free_list())
        self.free_all = torch.zeros(world * self.n_loc, dtype=torch.int32)
        self.fm = np.zeros((self.pcap + self.n, self.m))
        self.ga = np.array([cfg.ga.pc, cfg.ga.eta, cfg.ga.pm, cfg.ga.xi])

    def _free_list(self):
        return np.nonzero(~self.used)[0][: self.n_loc].astype(np.int32)

    def sync(self):
        pass

    def on_stream(self):
        import contextlib
        return contextlib.nullcontext()

    def pack(self, slots, row0=0):
        self.send_buf[row0: row0 + len(slots)] = torch.from_numpy(self.pool[np.asarray(slots, dtype=np.int64)])

    def reproduce(self, recv_pos, c_sbx, c_pm, unit_begin=0, unit_count=0):
        """Pairs [unit_begin, unit_begin + unit_count) of this rank (0: all), as GpuShard.reproduce."""
        u0, cnt = unit_begin, (unit_count or self.h_loc - unit_begin)
        recv_pos = np.asarray(recv_pos, dtype=np.int64)
        buf = self.recv_buf.numpy()
        pa = np.ascontiguousarray(buf[recv_pos[u0:u0 + cnt]])
        pb = np.ascontiguousarray(buf[recv_pos[self.h_loc + u0: self.h_loc + u0 + cnt]])
        ca, cb = np.empty_like(pa), np.empty_like(pb)
        _p, u64 = self._p, self.u64
        self.o.lib.to_reproduce_pairs(_p(pa), _p(pb), u64(cnt), u64(self.d), u64(self.rank * self.h_loc + u0), u64(self.n),
                                      u64(self.cfg.seed), u64(c_sbx), u64(c_pm), _p(self.ga), _p(self.lo), _p(self.hi), _p(ca), _p(cb))
        free = self.free_slot.numpy().astype(np.int64)
        f_loc = self.f_off_loc.numpy()
        for kids, first in ((ca, u0), (cb, self.h_loc + u0)):
            self.pool[free[first:first + cnt]] = kids
            f_loc[first:first + cnt] = self.o.evaluate(self.cfg.problem, kids, self.m)

    def place_f(self, P, initial):
        g = self.f_gather.numpy()
        if initial:
            self.fm[: self.n] = g
            return
        half = self.n // 2
        for rk in range(self.world):
            blk = g[rk * self.n_loc:(rk + 1) * self.n_loc]
            self.fm[P + rk * self.h_loc: P + (rk + 1) * self.h_loc] = blk[: self.h_loc]
            self.fm[P + half + rk * self.h_loc: P + half + (rk + 1) * self.h_loc] = blk[self.h_loc:]

    def select_local(self, P, lo, hi, t):
        rows = P + self.n
        sel = self.o.rv_select(self.fm[:rows], self.v, self.gamma, t, self.cfg.generations, self.cfg.alpha)
        self._assoc, self._apd = sel.assoc.astype(np.int64), sel.apd
        keys = np.full(self.r, np.iinfo(np.int64).max, dtype=np.int64)
        first = np.full(self.r, np.iinfo(np.int32).max, dtype=np.int32)
        k = (order_key(self._apd[lo:hi]) ^ KEY_FLIP).view(np.int64)  # signed, order preserving
        np.minimum.at(keys, self._assoc[lo:hi], k)
        np.minimum.at(first, self._assoc[lo:hi], ((np.arange(lo, hi, dtype=np.uint32)) ^ np.uint32(0x80000000)).view(np.int32))
        self.best_key.copy_(torch.from_numpy(keys))
        self.first_row.copy_(torch.from_numpy(first))

    def select_rows(self, lo, hi):
        keys = self.best_key.numpy()
        k = (order_key(self._apd[lo:hi]) ^ KEY_FLIP).view(np.int64)
        hit = k == keys[self._assoc[lo:hi]]
        best = np.full(self.r, np.iinfo(np.int32).max, dtype=np.int32)
        rows = ((np.arange(lo, hi, dtype=np.uint32)) ^ np.uint32(0x80000000)).view(np.int32)
        np.minimum.at(best, self._assoc[lo:hi][hit], rows[hit])
        self.best_row.copy_(torch.from_numpy(best))

    def select_finish(self):
        first = self.first_row.numpy().view(np.uint32) ^ np.uint32(0x80000000)
        best = self.best_row.numpy().view(np.uint32) ^ np.uint32(0x80000000)
        valid = first != np.uint32(0xffffffff)
        self._elite = best[valid].astype(np.uint32)
        return self._elite.copy()

    def commit(self, count, own_slots, t):
        self.fm[:count] = self.fm[self._elite.astype(np.int64)]
        self.used[:] = False
        self.used[np.asarray(own_slots, dtype=np.int64)] = True
        self.free_slot = torch.from_numpy(self._free_list())
        if (t + 1) % self.adapt_every == 0:
            f = self.fm[:count]
            self.v, self.gamma = self.o.adapt(self.v0, self.v, self.gamma, f.min(axis=0), f.max(axis=0))

    def free_slots_host(self):
        return self.free_all.numpy()


def _worker(rank, world, port, problem, n, d, m, gens, seed, out_dir, chunks):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      TEMO_B200_EXCHANGE_CHUNKS=str(chunks))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        import paper_2404_01159_b200 as tb
        from paper_2404_01159_b200.dist import ShardedRvea, TorchComm
        oracle = Oracle()
        cfg = tb.RunConfig(problem=problem, pop=n, dim=d, obj=m, generations=gens, seed=seed)
        shard = CpuShard(cfg, rank, world, oracle)
        run = ShardedRvea(cfg, TorchComm(), shard)
        pops, elites = [], []
        for _ in range(gens):
            pops.append(run.step())
            elites.append(run.last_elite.copy())
        idx, slots = run.own_slots()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pops=np.array(pops), idx=idx, x=shard.pool[slots.astype(np.int64)],
                 f=shard.fm[: run.P], v=shard.v, gamma=shard.gamma, counter=np.array([run.counter]),
                 elite_last=elites[-1], elite_first=elites[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("dtlz2", 24, 9, 3, 8, 7, 1), ("dtlz1", 40, 12, 3, 12, 3, 4), ("dtlz3", 16, 6, 2, 6, 11, 3),
                                  ("dtlz2", 36, 7, 3, 6, 5, 9)])
def test_sharded_orchestration_world2_matches_single_process(tmp_path, oracle, case):
    """The last field is the number of pieces the parent exchange is cut into (pipelined with reproduction): one piece,
    several, more pieces than some chunks have pairs."""
    problem, n, d, m, gens, seed, chunks = case
    world = 2
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(world, port, problem, n, d, m, gens, seed, str(tmp_path), chunks), nprocs=world, join=True)
    exp = oracle.rvea_run(problem, n, d, m, gens, seed=seed)
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for p in parts:  # replicated state is identical on every rank and equals the single-process run
        assert np.array_equal(p["pops"], exp["pop_size"])
        assert np.array_equal(p["f"], exp["f"])
        assert np.array_equal(p["v"], exp["v"]) and np.array_equal(p["gamma"], exp["gamma"])
        assert int(p["counter"][0]) == exp["counter"]
    # the sharded X (each rank holds the survivors born there) reassembles to the single-process population
    x = np.empty_like(exp["x"])
    seen = np.zeros(len(x), dtype=bool)
    for p in parts:
        x[p["idx"]] = p["x"]
        seen[p["idx"]] = True
    assert seen.all() and np.array_equal(x, exp["x"])


def test_shard_plan_is_consistent_across_ranks(oracle):
    """Every rank derives the same exchange from the replicated tables: what g sends to h is what h expects."""
    from paper_2404_01159_b200.dist import shard_plan
    n, d, world, P, seed, counter = 48, 5, 4, 37, 9, 1234
    rng = np.random.default_rng(0)
    owner = rng.integers(0, world, P).astype(np.int32)
    slot = rng.integers(0, 1000, P).astype(np.uint32)
    for chunks in (1, 2, 5):
        _check_plans(oracle, [shard_plan(seed, counter, P, n, d, r, world, owner, slot, chunks) for r in range(world)],
                     n, d, world, P, seed, counter, owner, slot, chunks)


def _check_plans(oracle, plans, n, d, world, P, seed, counter, owner, slot, chunks):
    pool_idx, c = oracle.parent_pool_indices(P, n, seed, counter)
    perm, c = oracle.shuffle_indices(seed, c, n)
    half, h_loc = n // 2, n // 2 // world
    for h in range(world):
        assert plans[h]["c_sbx"] == c and plans[h]["c_pm"] == c + 3 * half * d + half
        assert plans[h]["c_end"] == plans[h]["c_pm"] + 2 * n * d
        rows = [h * h_loc + j if j < h_loc else half + h * h_loc + (j - h_loc) for j in range(2 * h_loc)]
        want = pool_idx[perm[rows].astype(np.int64)].astype(np.int64)  # survivor index of every local mating row
        # rebuild the receive buffer of rank h from what every source says it sends, piece after piece
        recv = []
        per_chunk = -(-h_loc // chunks)
        for ch in range(chunks):
            first = len(recv)
            for g in range(world):
                sc = plans[g]["send_counts"].astype(np.int64)  # [chunks, world]
                start = int(sc[:ch].sum() + sc[ch, :h].sum())
                recv += [(g, int(s)) for s in plans[g]["send_slots"][start:start + int(sc[ch, h])]]
                assert int(plans[h]["recv_counts"][ch, g]) == int(sc[ch, h])
            # the parents of the pairs of piece ch are all inside piece ch
            for j in range(2 * h_loc):
                if (j % h_loc) // per_chunk == ch:
                    assert first <= int(plans[h]["recv_pos"][j]) < len(recv)
        for j, k in enumerate(want):
            assert recv[int(plans[h]["recv_pos"][j])] == (int(owner[k]), int(slot[k]))


def test_shard_plan_and_tables_large_threaded(oracle):
    """Sizes at which the host bookkeeping runs multi-threaded (one thread per destination / per survivor range):
    same consistency properties, and the table update equals a straightforward numpy transcription."""
    import ctypes as C
    from paper_2404_01159_b200 import _lib
    from paper_2404_01159_b200.dist import shard_plan, child_location
    n, d, world, P, seed, counter = 4 * 8192, 3, 4, 30011, 5, 77
    rng = np.random.default_rng(1)
    owner = rng.integers(0, world, P).astype(np.int32)
    slot = rng.integers(0, 50000, P).astype(np.uint32)
    for chunks in (1, 4):
        _check_plans(oracle, [shard_plan(seed, counter, P, n, d, r, world, owner, slot, chunks) for r in range(world)],
                     n, d, world, P, seed, counter, owner, slot, chunks)
    # survivor tables after a selection that keeps `count` rows of the merged population
    n, world, P, count, rank = 1 << 17, 4, 100000, 90000, 2
    n_loc = n // world
    owner = rng.integers(0, world, max(P, count)).astype(np.int32)
    slot = rng.integers(0, 1 << 20, max(P, count)).astype(np.uint32)
    elite = np.sort(rng.choice(P + n, count, replace=False)).astype(np.uint32)
    free_all = rng.integers(0, 1 << 20, world * n_loc).astype(np.uint32)
    exp_owner, exp_slot = np.empty(count, np.int32), np.empty(count, np.uint32)
    par = elite < P
    exp_owner[par], exp_slot[par] = owner[elite[par]], slot[elite[par]]
    rk, j = child_location(elite[~par].astype(np.int64) - P, n, world)
    exp_owner[~par], exp_slot[~par] = rk, free_all[rk.astype(np.int64) * n_loc + j]
    o, sl = owner.copy(), slot.copy()
    own = np.empty(count, dtype=np.uint32)
    own_count = C.c_uint64(0)
    u32p, i32p = C.POINTER(C.c_uint32), C.POINTER(C.c_int32)
    rc = _lib.load().temo_b200_shard_update_tables(elite.ctypes.data_as(u32p), C.c_uint64(count), C.c_uint64(P), C.c_uint64(n), rank, world,
                                                   free_all.ctypes.data_as(u32p), o.ctypes.data_as(i32p), sl.ctypes.data_as(u32p),
                                                   own.ctypes.data_as(u32p), C.byref(own_count))
    assert rc == 0
    assert np.array_equal(o[:count], exp_owner) and np.array_equal(sl[:count], exp_slot)
    assert np.array_equal(own[: own_count.value], exp_slot[exp_owner == rank])
