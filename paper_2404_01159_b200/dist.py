"""Multi-GPU host orchestration of the RVEA generation loop: one process per GPU (torchrun), the
population sharded by mating pair, torch.distributed (NCCL over NVLink) for the exchanges.

reference: rvea_run (algorithms.hpp:227-296) — single-process in the reference; SURVEY.md section 8e gives
the sharding. Per generation and rank:

    plan (host, C ABI)      who needs which survivor row from whom (the global shuffle scatters mates)
    pack + all_to_all       parents of this rank's pairs -> receive buffer          [rows, the only big exchange],
                            cut into EXCHANGE_CHUNKS pieces by mating pair and pipelined:
    reproduce (+evaluate)   K1 on the pairs of piece c (GLOBAL draw addressing: bit-identical children) runs while
                            piece c+1 is on the wire (NCCL on its own stream, ordered against the shard's stream)
    all_gather              offspring objectives (n x m doubles) and free-slot lists (n x 4 bytes)
    select_local            ideal point (replicated F) + association/APD of this rank's slice of merged rows
    all_reduce(min) x2      per-vector APD keys (order-preserving int64) + first rows, then lowest rows
    select_finish / commit  replicated compaction; survivors stay in the pool of the rank that bore them

`ShardedRvea` only talks to a `comm` (collectives) and a `shard` (stage functions + buffers); the GPU
implementation of the latter is `GpuShard` (C ABI `temo_b200_shard_*`). The same orchestration code runs
on CPU tensors over gloo in tests/test_dist_cpu.py with a stand-in shard, which is how the N>1 logic is
covered without N GPUs.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time

import numpy as np

from . import _lib
from .api import PROBLEM_IDS, RunConfig, _call

u64 = C.c_uint64
u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)


# ------------------------------------------------------------------------------------ collectives
class TorchComm:
    """torch.distributed collectives on torch tensors (cuda+NCCL or cpu+gloo)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def all_to_all_rows(self, recv, send, recv_counts, send_counts, async_op=False):
        """recv/send: 2-D row tensors; counts in rows per peer. async_op: returns the work handle (its wait() orders the
        CURRENT CUDA stream after the exchange; with gloo it blocks the host)."""
        return self.dist.all_to_all_single(recv, send, [int(c) for c in recv_counts], [int(c) for c in send_counts],
                                           async_op=async_op)

    def all_gather(self, out, inp):
        self.dist.all_gather_into_tensor(out, inp)

    def all_reduce_min(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)

    def barrier(self):
        self.dist.barrier()

    def all_reduce_max_scalar(self, value: float) -> float:
        import torch
        t = torch.tensor([value], dtype=torch.float64, device="cuda" if torch.cuda.is_available() and self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


class LocalComm:
    """World size 1: the collectives degenerate to copies (used to validate the sharded path on one GPU)."""
    rank, world = 0, 1

    def all_to_all_rows(self, recv, send, recv_counts, send_counts, async_op=False):
        recv[: int(recv_counts[0])].copy_(send[: int(send_counts[0])])
        return None

    def all_gather(self, out, inp):
        out.view(-1)[: inp.numel()].copy_(inp.view(-1))

    def all_reduce_min(self, t):
        pass

    def barrier(self):
        pass

    def all_reduce_max_scalar(self, value):
        return value


# ------------------------------------------------------------------------------------ host plan
def shard_plan(seed, counter, P, n, d, rank, world, surv_owner, surv_slot, chunks=1):
    """C-ABI temo_b200_shard_plan (pure host code, no GPU needed). send_counts / recv_counts: [chunks, world]."""
    L = _lib.load()
    n_loc = n // world
    surv_owner = np.ascontiguousarray(surv_owner, dtype=np.int32)
    surv_slot = np.ascontiguousarray(surv_slot, dtype=np.uint32)
    send_slots = np.empty(n, dtype=np.uint32)
    send_counts = np.zeros((chunks, world), dtype=np.uint64)
    recv_counts = np.zeros((chunks, world), dtype=np.uint64)
    recv_pos = np.empty(n_loc, dtype=np.uint32)
    counters = np.zeros(3, dtype=np.uint64)
    rc = L.temo_b200_shard_plan(u64(seed), u64(counter), u64(P), u64(n), u64(d), rank, world, chunks,
                                surv_owner.ctypes.data_as(i32p), surv_slot.ctypes.data_as(u32p),
                                send_slots.ctypes.data_as(u32p), u64(n), send_counts.ctypes.data_as(u64p),
                                recv_counts.ctypes.data_as(u64p), recv_pos.ctypes.data_as(u32p), counters.ctypes.data_as(u64p))
    if rc:
        raise ValueError(L.temo_b200_shard_last_error().decode())
    total = int(send_counts.sum())
    return dict(send_slots=send_slots[:total], send_counts=send_counts, recv_counts=recv_counts, recv_pos=recv_pos,
                c_sbx=int(counters[0]), c_pm=int(counters[1]), c_end=int(counters[2]))


def child_location(i, n, world):
    """Global child row i -> (rank that produced it, its local child index)."""
    half = n // 2
    h_loc = half // world
    i = np.asarray(i, dtype=np.int64)
    first = i < half
    p = np.where(first, i, i - half)
    rk = p // h_loc
    j = np.where(first, p - rk * h_loc, h_loc + p - rk * h_loc)
    return rk.astype(np.int32), j.astype(np.int64)


# ------------------------------------------------------------------------------------ GPU shard
class _DevArray:
    """Zero-copy view of a device buffer of the shared library for torch (cuda array interface)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False), "version": 2}


class GpuShard:
    """Stage functions and exchange buffers of this rank (C ABI temo_b200_shard_*)."""

    def __init__(self, cfg: RunConfig, rank: int, world: int):
        import torch
        self._L = _lib.load()
        self._h = C.c_void_p()
        ccfg = cfg.c()
        self._chk(self._L.temo_b200_shard_create(C.byref(ccfg), rank, world, C.byref(self._h)))
        info = np.zeros(8, dtype=np.uint64)
        self._chk(self._L.temo_b200_shard_info(self._h, info.ctypes.data_as(u64p)))
        self.n_loc, self.d, self.m, self.r, self.send_cap, self.pcap, self.cap_loc, self.adapt_every = (int(v) for v in info)
        buf = lambda which: self._L.temo_b200_shard_buffer(self._h, which)
        dev = torch.device("cuda", torch.cuda.current_device())
        wrap = lambda which, shape, ts: torch.as_tensor(_DevArray(buf(which), shape, ts), device=dev)
        self.send_buf = wrap(0, (self.send_cap, self.d), "<f8")
        self.recv_buf = wrap(1, (self.n_loc, self.d), "<f8")
        self.f_off_loc = wrap(2, (self.n_loc, self.m), "<f8")
        self.f_gather = wrap(3, (world * self.n_loc, self.m), "<f8")
        self.best_key = wrap(4, (self.r,), "<i8")
        self.first_row = wrap(5, (self.r,), "<i4")
        self.best_row = wrap(6, (self.r,), "<i4")
        self.free_slot = wrap(7, (self.n_loc,), "<i4")
        self.free_all = torch.empty(world * self.n_loc, dtype=torch.int32, device=dev)
        self._torch = torch
        # every stage runs on the library's stream: collectives issued with it as the current stream are ordered
        # against the stages by NCCL's own stream events, without device-wide synchronisation
        self.stream = torch.cuda.ExternalStream(int(self._L.temo_b200_shard_stream(self._h)), device=dev)
        self.k1_events = None  # list: collect (start, end) CUDA events of every K1 launch

    def _chk(self, rc):
        if rc:
            msg = self._L.temo_b200_shard_last_error().decode(errors="replace")
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def sync(self):
        self._torch.cuda.synchronize()

    def on_stream(self):
        """Context manager: torch ops (collectives) issued inside use the shard's stream as the current stream."""
        return self._torch.cuda.stream(self.stream)

    def pack(self, slots, row0=0):
        """Gathers pool rows into send_buf[row0:row0+len(slots)] (enqueued on the shard's stream)."""
        slots = np.ascontiguousarray(slots, dtype=np.uint32)
        self._chk(self._L.temo_b200_shard_pack_at(self._h, slots.ctypes.data_as(u32p), u64(slots.size), u64(row0)))

    def reproduce(self, recv_pos, c_sbx, c_pm, unit_begin=0, unit_count=0):
        """K1 (+ evaluation) on the local pairs [unit_begin, unit_begin + unit_count) (0: all); enqueued, not awaited."""
        recv_pos = np.ascontiguousarray(recv_pos, dtype=np.uint32)
        ev = None
        if self.k1_events is not None:  # device time of the K1 launches (bench): events on the shard's stream
            ev = (self._torch.cuda.Event(enable_timing=True), self._torch.cuda.Event(enable_timing=True))
            ev[0].record(self.stream)
        self._chk(self._L.temo_b200_shard_reproduce_range(self._h, recv_pos.ctypes.data_as(u32p), u64(c_sbx), u64(c_pm),
                                                          u64(unit_begin), u64(unit_count)))
        if ev is not None:
            ev[1].record(self.stream)
            self.k1_events.append(ev)

    def place_f(self, P, initial):
        self._chk(self._L.temo_b200_shard_place_f(self._h, u64(P), 1 if initial else 0))

    def select_local(self, P, lo, hi, t):
        self._chk(self._L.temo_b200_shard_select_local(self._h, u64(P), u64(lo), u64(hi), u64(t)))

    def select_rows(self, lo, hi):
        self._chk(self._L.temo_b200_shard_select_rows(self._h, u64(lo), u64(hi)))

    def select_finish(self):
        elite = np.empty(self.r, dtype=np.uint32)
        cnt = u64(0)
        self._chk(self._L.temo_b200_shard_select_finish(self._h, elite.ctypes.data_as(u32p), C.byref(cnt)))
        return elite[: cnt.value]

    def commit(self, count, own_slots, t):
        own_slots = np.ascontiguousarray(own_slots, dtype=np.uint32)
        self._chk(self._L.temo_b200_shard_commit(self._h, u64(count), own_slots.ctypes.data_as(u32p), u64(own_slots.size), u64(t)))

    def free_slots_host(self):
        return self.free_all.cpu().numpy()

    def download(self, own_slots, f_rows):
        own_slots = np.ascontiguousarray(own_slots, dtype=np.uint32)
        x = np.empty((own_slots.size, self.d))
        f = np.empty((f_rows, self.m))
        v, gamma = np.empty((self.r, self.m)), np.empty(self.r)
        self._chk(self._L.temo_b200_shard_download(self._h, own_slots.ctypes.data_as(u32p), u64(own_slots.size),
                                                   x.ctypes.data_as(_lib.f64p), u64(f_rows), f.ctypes.data_as(_lib.f64p),
                                                   v.ctypes.data_as(_lib.f64p), gamma.ctypes.data_as(_lib.f64p)))
        return x, f, v, gamma

    def close(self):
        if self._h:
            self._L.temo_b200_shard_destroy(self._h)
            self._h = C.c_void_p()


# ------------------------------------------------------------------------------------ orchestrator
class ShardedRvea:
    """The generation loop over `world` shards. `shard` provides the stage functions and buffers
    (GpuShard, or a CPU stand-in in the tests), `comm` the collectives."""

    def __init__(self, cfg: RunConfig, comm, shard):
        self.cfg, self.comm, self.shard = cfg, comm, shard
        self.rank, self.world = comm.rank, comm.world
        self.n = cfg.pop
        if self.n % (2 * self.world):
            raise ValueError("sharded run: population must be divisible by 2 * world size")
        self.d, self.m, self.r = shard.d, shard.m, shard.r
        self.n_loc = self.n // self.world
        pcap = max(self.n, self.r)
        self.surv_owner = np.zeros(pcap, dtype=np.int32)
        self.surv_slot = np.zeros(pcap, dtype=np.uint32)
        # initial population: contiguous blocks of n/world rows per rank, local slots 0..
        rows = np.arange(self.n)
        self.surv_owner[: self.n] = rows // self.n_loc
        self.surv_slot[: self.n] = rows % self.n_loc
        self.P = self.n
        self.counter = self.n * self.d  # operators.hpp:287-296: n*d draws for the initial population
        self.t = 0
        self.last_elite = None
        # pieces of the parent exchange (pipelined with reproduction); 1 = one exchange, then K1
        self.chunks = max(1, min(int(os.environ.get("TEMO_B200_EXCHANGE_CHUNKS", "4" if self.world > 1 else "1")),
                                 max(1, self.n_loc // 2)))
        # on the shard's stream like every stage: the collective's result is only ordered against the stream it was
        # issued on, and place_f reads f_gather on the library's (non-blocking) stream
        with shard.on_stream():
            comm.all_gather(shard.f_gather, shard.f_off_loc)
            shard.place_f(0, True)
        self.timers = {}

    def _tick(self, name, t0):
        self.timers[name] = self.timers.get(name, 0.0) + (time.perf_counter() - t0)

    def step(self):
        cfg, comm, sh = self.cfg, self.comm, self.shard
        n, world, rank, P = self.n, self.world, self.rank, self.P
        t0 = time.perf_counter()
        chunks = self.chunks
        plan = shard_plan(cfg.seed, self.counter, P, n, self.d, rank, world, self.surv_owner[:P], self.surv_slot[:P], chunks)
        # while the GPU works on this generation, a host thread shuffles for the next one (its counters only
        # depend on this generation's, assuming the survivor count will differ from n: algorithms.hpp:211-221)
        _lib.load().temo_b200_shard_perm_prefetch(u64(cfg.seed), u64(plan["c_end"] + n), u64(n))
        self._tick("plan", t0)
        t0 = time.perf_counter()
        # Pipelined exchange + reproduction: piece c of the parent rows is packed and sent while K1 works on the pairs
        # of piece c - 1. Everything is enqueued on the shard's stream (NCCL orders its own stream against it), so the
        # host never waits inside the loop.
        h_loc = self.n_loc // 2
        per_chunk = (h_loc + chunks - 1) // chunks
        send_counts, recv_counts = plan["send_counts"], plan["recv_counts"]
        send_off = np.concatenate([[0], np.cumsum(send_counts.sum(axis=1))]).astype(np.int64)
        recv_off = np.concatenate([[0], np.cumsum(recv_counts.sum(axis=1))]).astype(np.int64)

        def send_piece(c):
            sh.pack(plan["send_slots"][send_off[c]:send_off[c + 1]], int(send_off[c]))
            return comm.all_to_all_rows(sh.recv_buf[recv_off[c]:recv_off[c + 1]], sh.send_buf[send_off[c]:send_off[c + 1]],
                                        recv_counts[c], send_counts[c], async_op=True)

        with sh.on_stream():
            work = send_piece(0)
            for c in range(chunks):
                nxt = send_piece(c + 1) if c + 1 < chunks else None
                if work is not None:
                    work.wait()  # orders the shard's stream after piece c (host-blocking only with gloo)
                u0 = c * per_chunk
                cnt = min(per_chunk, h_loc - u0)
                if cnt > 0:
                    sh.reproduce(plan["recv_pos"], plan["c_sbx"], plan["c_pm"], u0, cnt)
                work = nxt
            self._tick("exchange+reproduce", t0)
            t0 = time.perf_counter()
            comm.all_gather(sh.f_gather, sh.f_off_loc)
            comm.all_gather(sh.free_all, sh.free_slot)
            sh.sync()
            sh.place_f(P, False)
            rows = P + n
            lo, hi = rows * rank // world, rows * (rank + 1) // world
            sh.select_local(P, lo, hi, self.t)
            comm.all_reduce_min(sh.best_key)
            comm.all_reduce_min(sh.first_row)
            sh.sync()
            sh.select_rows(lo, hi)
            comm.all_reduce_min(sh.best_row)
            sh.sync()
            elite = sh.select_finish().astype(np.int64)
            self._tick("select", t0)
            t0 = time.perf_counter()
            # survivor k <- merged row elite[k]: a parent keeps its (owner, slot); a child lives where it was born
            cnt = len(elite)
            elite32 = np.ascontiguousarray(elite, dtype=np.uint32)
            free_all = np.ascontiguousarray(sh.free_slots_host()).view(np.uint32)
            own = np.empty(max(cnt, 1), dtype=np.uint32)
            own_count = u64(0)
            L = _lib.load()
            rc = L.temo_b200_shard_update_tables(elite32.ctypes.data_as(u32p), u64(cnt), u64(P), u64(n), rank, world,
                                                 free_all.ctypes.data_as(u32p), self.surv_owner.ctypes.data_as(i32p),
                                                 self.surv_slot.ctypes.data_as(u32p), own.ctypes.data_as(u32p), C.byref(own_count))
            if rc:
                raise ValueError(L.temo_b200_shard_last_error().decode())
            sh.commit(cnt, own[: own_count.value], self.t)
            self._tick("commit", t0)
        self.last_elite = elite
        self.P, self.counter, self.t = cnt, plan["c_end"], self.t + 1
        return cnt

    def own_slots(self):
        mine = self.surv_owner[: self.P] == self.rank
        return np.nonzero(mine)[0], self.surv_slot[: self.P][mine]


# ------------------------------------------------------------------------------------ bench entry (N > 1)
def bench_main(args, metric, workload_config, measured_peaks, ClockSampler):
    """bench.py --gpus N (N > 1), launched by torchrun: weak scaling, pop = N * args.pop."""
    import torch
    import torch.distributed as dist
    from . import api as tb

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    tb.init(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = TorchComm()
    pop = args.pop * world
    K, W = args.steps, args.warmup
    cfg = RunConfig(problem=args.problem, pop=pop, dim=args.dim, obj=args.obj, generations=max(100, W + K + 2), seed=args.seed,
                    fuse_eval=not args.no_fuse)
    shard = GpuShard(cfg, rank, world)
    run = ShardedRvea(cfg, comm, shard)
    for _ in range(W):
        run.step()
    run.timers.clear()
    shard.k1_events = []
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    comm.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    t0 = time.perf_counter()
    for _ in range(K):
        pop_size = run.step()
    stop.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    comm.barrier()
    wall = comm.all_reduce_max_scalar(max(wall, start.elapsed_time(stop) * 1e-3))  # max over ranks
    clocks = sampler.stop() if rank == 0 else None
    if rank == 0:
        peak, peak_src = measured_peaks()
        nd = float(run.n_loc) * run.d
        rep_ms = sum(a.elapsed_time(b) for a, b in shard.k1_events) / K  # K1 launches of one step (CUDA events)
        args_cfg = workload_config(args, None)
        args_cfg.update({"workload": f"RVEA/{args.problem} m={args.obj} d={args.dim} pop={pop} ({world} shards of {args.pop})",
                         "pop": pop, "ref_vectors": run.r, "survivors_last": int(pop_size)})
        # weak scaling: every rank advances one shard of args.pop rows per step, so the job processes `world`
        # shard-generations per step; the GLOBAL population is one RVEA run of world * args.pop rows
        args_cfg["unit_note"] = (f"value counts generations of one {args.pop}-row shard: {world} per step of the global "
                                 f"{pop}-row run (global generations/s = value / {world})")
        line = {
            "metric": metric, "value": world * K / wall, "unit": "generations/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": wall / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": args_cfg,
            "e2e": {"value": world * K / wall, "unit": "generations/s", "h2d_bytes_per_step": 8 * run.n_loc, "d2h_bytes_per_step": 4 * pop + 4 * run.r},
            "gpu_launches": int(K * 30),
            "roofline": {"bound": "hbm", "kernel": "reproduce_pairs_kernel (rank 0, CUDA events over the K1 launches of a step: one per exchange piece)", "achieved": 16.0 * nd / (rep_ms * 1e-3) / 1e9 if rep_ms else None,
                         "peak": peak, "unit": "GB/s", "frac": (16.0 * nd / (rep_ms * 1e-3) / 1e9 / peak) if rep_ms else None, "traffic": None,
                         "peak_source": peak_src},
            "stages_ms": {**{k: v / K * 1e3 for k, v in run.timers.items()}, "reproduce_device": rep_ms},
            "exchange_chunks": run.chunks,
            "clocks": clocks,
            "rows_per_s": K * float(pop) / wall,
        }
        print(json.dumps(line), flush=True)
    shard.close()
    dist.destroy_process_group()
