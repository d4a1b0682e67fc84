"""CPU, world_size 2 and 4 (gloo): the multi-GPU host orchestration (paper_2404_01159_b200.dist.ShardedRvea with
TorchComm) — stage order, objective / free-slot all-gathers, packed min-allreduces — driven end to end with a CPU
stand-in for the per-rank stage functions (the oracle does the arithmetic here; on the GPU it is GpuShard, whose
N > 1 device logic is covered on one GPU by tests/test_gpu_parity.py::test_sharded_world_n_on_one_gpu_*). The sharded
run must reproduce the single-process oracle run bit for bit: same survivor sets, same X, same F, every generation.
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
    """Stand-in for GpuShard: same stage functions and buffers (CPU tensors), arithmetic by the oracle. The peers'
    pools are not mapped but fetched (an all-gather of the small test pools inside reproduce), which is what the NVLink
    peer loads of K1 amount to; tables, counters and the generation live in the shard as in csrc/shard.cu."""

    def __init__(self, cfg, rank, world, oracle):
        from oracle.pyoracle import _p, u64
        self._p, self.u64 = _p, u64
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
        self.adapt_every = max(1, int(np.ceil(cfg.fr * cfg.generations)))
        self.lo_b, self.hi_b = oracle.problem_bounds(cfg.problem, self.d, self.m)
        self.pool = torch.zeros(self.cap_loc, self.d, dtype=torch.float64)
        rows0 = self.n_loc
        x, _ = oracle.random_reproduce(rows0, self.d, cfg.seed, rank * rows0 * self.d, self.lo_b, self.hi_b)
        self.pool[:rows0] = torch.from_numpy(x)
        self.used = np.zeros(self.cap_loc, dtype=bool)
        self.used[:rows0] = True
        self.f_off_loc = torch.from_numpy(oracle.evaluate(cfg.problem, x, self.m).copy())
        self.f_gather = torch.zeros(world * self.n_loc, self.m, dtype=torch.float64)
        self.best_key = torch.zeros(self.r, dtype=torch.int64)
        self.first_row = torch.zeros(self.r, dtype=torch.int32)
        self.best_row = torch.zeros(self.r, dtype=torch.int32)
        self.free_slot = torch.from_numpy(self._free_list())
        self.free_all = torch.zeros(world * self.n_loc, dtype=torch.int32)
        self.fm = np.zeros((self.pcap + self.n, self.m))
        self.ga = np.array([cfg.ga.pc, cfg.ga.eta, cfg.ga.pm, cfg.ga.xi])
        rows = np.arange(self.n)
        self.owner = (rows // self.n_loc).astype(np.int64)   # replicated survivor tables
        self.slot = (rows % self.n_loc).astype(np.int64)
        self.P, self.counter, self.t = self.n, self.n * self.d, 0
        self.comm = None

    def _free_list(self):
        return np.nonzero(~self.used)[0][: self.n_loc].astype(np.int32)

    def state(self):
        return dict(P=self.P, counter=self.counter, t=self.t, lo=getattr(self, "lo", 0), hi=getattr(self, "hi", 0))

    def sync(self):
        pass

    def on_stream(self):
        import contextlib
        return contextlib.nullcontext()

    def connect_peers(self, comm):
        self.comm = comm

    def place_initial_f(self):
        self.fm[: self.n] = self.f_gather.numpy()

    def begin(self):
        n, half, h_loc = self.n, self.n // 2, self.h_loc
        pool_idx, c = self.o.parent_pool_indices(self.P, n, self.cfg.seed, self.counter)
        perm, c = self.o.shuffle_indices(self.cfg.seed, c, n)
        self.c_sbx, self.c_pm = c, c + 3 * half * self.d + half
        self.c_end = self.c_pm + 2 * n * self.d
        rows = np.array([self.rank * h_loc + j if j < h_loc else half + self.rank * h_loc + (j - h_loc) for j in range(2 * h_loc)])
        k = pool_idx[perm[rows].astype(np.int64)].astype(np.int64)   # survivor index of every local mating row
        self._parent = (self.owner[k], self.slot[k])
        total = self.P + n
        self.lo, self.hi = total * self.rank // self.world, total * (self.rank + 1) // self.world

    def reproduce(self):
        pools = torch.zeros(self.world * self.cap_loc, self.d, dtype=torch.float64)
        self.comm.all_gather(pools, self.pool)   # the peers' pools (mapped, not copied, on the GPU)
        self.comm.calls -= 1
        pools = pools.numpy().reshape(self.world, self.cap_loc, self.d)
        own, sl = self._parent
        cnt = self.h_loc
        pa = np.ascontiguousarray(pools[own[:cnt], sl[:cnt]])
        pb = np.ascontiguousarray(pools[own[cnt:], sl[cnt:]])
        ca, cb = np.empty_like(pa), np.empty_like(pb)
        _p, u64 = self._p, self.u64
        self.o.lib.to_reproduce_pairs(_p(pa), _p(pb), u64(cnt), u64(self.d), u64(self.rank * self.h_loc), u64(self.n),
                                      u64(self.cfg.seed), u64(self.c_sbx), u64(self.c_pm), _p(self.ga), _p(self.lo_b), _p(self.hi_b),
                                      _p(ca), _p(cb))
        free = self.free_slot.numpy().astype(np.int64)
        f_loc = self.f_off_loc.numpy()
        pool = self.pool.numpy()
        for kids, first in ((ca, 0), (cb, self.h_loc)):
            pool[free[first:first + cnt]] = kids
            f_loc[first:first + cnt] = self.o.evaluate(self.cfg.problem, kids, self.m)

    def select_local(self):
        P, lo, hi = self.P, self.lo, self.hi
        g = self.f_gather.numpy()
        half = self.n // 2
        for rk in range(self.world):
            blk = g[rk * self.n_loc:(rk + 1) * self.n_loc]
            self.fm[P + rk * self.h_loc: P + (rk + 1) * self.h_loc] = blk[: self.h_loc]
            self.fm[P + half + rk * self.h_loc: P + half + (rk + 1) * self.h_loc] = blk[self.h_loc:]
        rows = P + self.n
        sel = self.o.rv_select(self.fm[:rows], self.v, self.gamma, self.t, self.cfg.generations, self.cfg.alpha)
        self._assoc, self._apd = sel.assoc.astype(np.int64), sel.apd
        keys = np.full(self.r, np.iinfo(np.int64).max, dtype=np.int64)
        first = np.full(self.r, np.iinfo(np.int32).max, dtype=np.int32)
        k = (order_key(self._apd[lo:hi]) ^ KEY_FLIP).view(np.int64)  # signed, order preserving
        np.minimum.at(keys, self._assoc[lo:hi], k)
        np.minimum.at(first, self._assoc[lo:hi], ((np.arange(lo, hi, dtype=np.uint32)) ^ np.uint32(0x80000000)).view(np.int32))
        self.best_key.copy_(torch.from_numpy(keys))
        self.first_row.copy_(torch.from_numpy(first))

    def select_rows(self):
        lo, hi = self.lo, self.hi
        keys = self.best_key.numpy()
        k = (order_key(self._apd[lo:hi]) ^ KEY_FLIP).view(np.int64)
        hit = k == keys[self._assoc[lo:hi]]
        best = np.full(self.r, np.iinfo(np.int32).max, dtype=np.int32)
        rows = ((np.arange(lo, hi, dtype=np.uint32)) ^ np.uint32(0x80000000)).view(np.int32)
        np.minimum.at(best, self._assoc[lo:hi][hit], rows[hit])
        self.best_row.copy_(torch.from_numpy(best))

    def finish(self):
        from paper_2404_01159_b200.dist import child_location
        first = self.first_row.numpy().view(np.uint32) ^ np.uint32(0x80000000)
        best = self.best_row.numpy().view(np.uint32) ^ np.uint32(0x80000000)
        valid = first != np.uint32(0xffffffff)
        elite = best[valid].astype(np.int64)
        self.last_elite = elite.copy()
        count, P, n = len(elite), self.P, self.n
        # survivor k <- merged row elite[k]: a parent keeps its (owner, slot); a child lives where it was born
        free_all = self.free_all.numpy().astype(np.int64)
        par = elite < P
        own, sl = np.empty(count, np.int64), np.empty(count, np.int64)
        own[par], sl[par] = self.owner[elite[par]], self.slot[elite[par]]
        rk, j = child_location(elite[~par] - P, n, self.world)
        own[~par], sl[~par] = rk, free_all[rk.astype(np.int64) * self.n_loc + j]
        self.owner, self.slot = own, sl
        self.fm[:count] = self.fm[elite]
        self.used[:] = False
        self.used[sl[own == self.rank]] = True
        self.free_slot.copy_(torch.from_numpy(self._free_list()))
        if (self.t + 1) % self.adapt_every == 0:
            f = self.fm[:count]
            self.v, self.gamma = self.o.adapt(self.v0, self.v, self.gamma, f.min(axis=0), f.max(axis=0))
        self.P, self.counter, self.t = count, self.c_end, self.t + 1
        return count


def _worker(rank, world, port, problem, n, d, m, gens, seed, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        import paper_2404_01159_b200 as tb
        from paper_2404_01159_b200.dist import ShardedRvea, TorchComm
        oracle = Oracle()
        cfg = tb.RunConfig(problem=problem, pop=n, dim=d, obj=m, generations=gens, seed=seed)
        shard = CpuShard(cfg, rank, world, oracle)
        comm = TorchComm()
        run = ShardedRvea(cfg, comm, shard)
        pops, elites = [], []
        for _ in range(gens):
            pops.append(run.step())
            elites.append(shard.last_elite.copy())
        mine = shard.owner == rank
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pops=np.array(pops), idx=np.nonzero(mine)[0],
                 x=shard.pool.numpy()[shard.slot[mine]], f=shard.fm[: run.P], v=shard.v, gamma=shard.gamma,
                 counter=np.array([run.counter]), elite_last=elites[-1], elite_first=elites[0],
                 collectives=np.array([comm.calls]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("dtlz2", 24, 9, 3, 8, 7, 2), ("dtlz1", 40, 12, 3, 12, 3, 2), ("dtlz3", 16, 6, 2, 6, 11, 2),
                                  ("dtlz2", 36, 7, 3, 6, 5, 2), ("dtlz2", 48, 10, 3, 6, 9, 4)])
def test_sharded_orchestration_matches_single_process(tmp_path, oracle, case):
    """World size 2 and 4 over gloo: the orchestration (stage order, the five collectives per generation, the packed
    order-preserving keys of the min-allreduces) reproduces the single-process oracle run bit for bit."""
    problem, n, d, m, gens, seed, world = case
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(world, port, problem, n, d, m, gens, seed, str(tmp_path)), nprocs=world, join=True)
    exp = oracle.rvea_run(problem, n, d, m, gens, seed=seed)
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for p in parts:  # replicated state is identical on every rank and equals the single-process run
        assert np.array_equal(p["pops"], exp["pop_size"])
        assert np.array_equal(p["f"], exp["f"])
        assert np.array_equal(p["v"], exp["v"]) and np.array_equal(p["gamma"], exp["gamma"])
        assert int(p["counter"][0]) == exp["counter"]
        assert int(p["collectives"][0]) == 1 + 5 * gens  # init all-gather + two all-gathers and three min-allreduces per generation
    # the sharded X (each rank holds the survivors born there) reassembles to the single-process population
    x = np.empty_like(exp["x"])
    seen = np.zeros(len(x), dtype=bool)
    for p in parts:
        x[p["idx"]] = p["x"]
        seen[p["idx"]] = True
    assert seen.all() and np.array_equal(x, exp["x"])


def test_child_location_and_key_packing():
    """Host helpers of the sharded path: where a child row lives, and the order-preserving packing the min-allreduces
    rely on (signed int64 view of an APD key, signed int32 view of a row with 0xffffffff = none staying the maximum)."""
    from paper_2404_01159_b200.dist import child_location
    n, world = 48, 4
    half, h_loc = n // 2, n // 2 // world
    rk, j = child_location(np.arange(n), n, world)
    for i in range(n):
        p = i if i < half else i - half
        assert rk[i] == p // h_loc and j[i] == (p % h_loc if i < half else h_loc + p % h_loc)
    x = np.array([0.0, 1e-300, 1.0, 2.5, 1e300, np.inf])
    k = (order_key(x) ^ KEY_FLIP).view(np.int64)
    assert np.all(np.diff(k) > 0)
    rows = np.array([0, 1, 77, 0x7fffffff, 0xfffffffe, 0xffffffff], dtype=np.uint32)
    sr = (rows ^ np.uint32(0x80000000)).view(np.int32)
    assert np.all(np.diff(sr.astype(np.int64)) > 0)
