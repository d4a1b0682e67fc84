"""Multi-GPU host orchestration of the RVEA generation loop: one process per GPU (torchrun), the
population sharded by mating pair, torch.distributed (NCCL over NVLink) for the small exchanges.

reference: rvea_run (algorithms.hpp:227-296) — single-process in the reference; SURVEY.md section 8e gives
the sharding. Per generation and rank (csrc/shard.cu has the stage functions):

    begin                   draw counters, mating permutation (4 n bytes H2D), one parent ADDRESS per local mating row
                            from the device-resident survivor -> (owner rank, slot) tables
    reproduce (+evaluate)   K1 on this rank's pairs; parents are streamed straight out of the peers' pools, which every
                            rank maps once through CUDA IPC (NVLink peer loads inside the kernel: no pack, no all-to-all)
    all_gather x2           offspring objectives (n x m doubles) and free-slot lists (n x 4 bytes)
    select_local            ideal point (replicated F) + association/APD of this rank's slice of merged rows
    all_reduce(min) x2      per-vector APD keys (order-preserving int64) + first rows
    select_rows
    all_reduce(min)         lowest rows attaining the minimum
    finish                  replicated compaction, survivor tables, free list, adaptation; the survivor count comes back
                            to the host (the one synchronisation of a generation)

`ShardedRvea` only talks to a `comm` (collectives) and a `shard` (stage functions + buffers); the GPU
implementation of the latter is `GpuShard` (C ABI `temo_b200_shard_*`). The same orchestration code runs
on CPU tensors over gloo in tests/test_dist_cpu.py with a stand-in shard, and in-process with several GpuShards
of one GPU (ThreadComm), which is how the N>1 logic is covered without N GPUs.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import threading
import time

import numpy as np

from . import _lib
from .api import RunConfig

u64 = C.c_uint64
u64p = C.POINTER(C.c_uint64)


# ------------------------------------------------------------------------------------ collectives
class TorchComm:
    """torch.distributed collectives on torch tensors (cuda+NCCL or cpu+gloo)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.calls = 0

    def _staged(self, t):
        """gloo has no CUDA collectives: device tensors go through the host (tests on one GPU; NCCL takes them as they are)."""
        return t.is_cuda and self.dist.get_backend() == "gloo"

    def all_gather(self, out, inp):
        self.calls += 1
        if self._staged(inp):
            host = out.cpu()
            self.dist.all_gather_into_tensor(host, inp.cpu())
            out.copy_(host)
            return
        self.dist.all_gather_into_tensor(out, inp)

    def all_reduce_min(self, t):
        self.calls += 1
        if self._staged(t):
            host = t.cpu()
            self.dist.all_reduce(host, op=self.dist.ReduceOp.MIN)
            t.copy_(host)
            return
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)

    def all_gather_bytes(self, payload) -> list:
        """Host-side exchange of small blobs (the IPC handles of the pools)."""
        out = [None] * self.world
        self.dist.all_gather_object(out, payload)
        return out

    def barrier(self):
        self.dist.barrier()

    def all_reduce_max_scalar(self, value: float) -> float:
        import torch
        t = torch.tensor([value], dtype=torch.float64, device="cuda" if torch.cuda.is_available() and self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


class LocalComm:
    """World size 1: the collectives degenerate to copies (validates the sharded path on one GPU)."""
    rank, world = 0, 1

    def __init__(self):
        self.calls = 0

    def all_gather(self, out, inp):
        self.calls += 1
        out.view(-1)[: inp.numel()].copy_(inp.view(-1))

    def all_reduce_min(self, t):
        self.calls += 1

    def all_gather_bytes(self, payload):
        return [payload]

    def barrier(self):
        pass

    def all_reduce_max_scalar(self, value):
        return value


class ThreadComm:
    """`world` ranks as threads of ONE process (each with its own shard on the same GPU): the collectives meet at a
    barrier and combine the participants' tensors. Test vehicle for the N > 1 device logic on a single GPU."""

    class Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self.s, self.rank, self.world, self.calls = shared, rank, shared.world, 0

    def _exchange(self, item):
        self.s.slots[self.rank] = item
        self.s.barrier.wait()
        items = list(self.s.slots)
        self.s.barrier.wait()
        return items

    def all_gather(self, out, inp):
        import torch
        self.calls += 1
        torch.cuda.synchronize()
        items = self._exchange(inp)
        flat = out.view(-1)
        k = inp.numel()
        for g, t in enumerate(items):
            flat[g * k:(g + 1) * k].copy_(t.view(-1))
        torch.cuda.synchronize()
        self.s.barrier.wait()

    def all_reduce_min(self, t):
        import torch
        self.calls += 1
        torch.cuda.synchronize()
        items = self._exchange(t)
        red = torch.stack(list(items)).min(dim=0).values
        torch.cuda.synchronize()
        self.s.barrier.wait()
        t.copy_(red)
        torch.cuda.synchronize()
        self.s.barrier.wait()

    def all_gather_bytes(self, payload):
        return self._exchange(payload)

    def barrier(self):
        self.s.barrier.wait()

    def all_reduce_max_scalar(self, value):
        return max(self._exchange(value))


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

    def __init__(self, cfg: RunConfig, rank: int, world: int, direct_peers: bool = False):
        import torch
        self._L = _lib.load()
        self._h = C.c_void_p()
        self.rank, self.world = rank, world
        ccfg = cfg.c()
        self._chk(self._L.temo_b200_shard_create(C.byref(ccfg), rank, world, C.byref(self._h)))
        info = self._info()
        self.n_loc, self.d, self.m, self.r, self.pcap, self.cap_loc, self.adapt_every = (int(v) for v in info[:7])
        buf = lambda which: self._L.temo_b200_shard_buffer(self._h, which)
        dev = torch.device("cuda", torch.cuda.current_device())
        wrap = lambda which, shape, ts: torch.as_tensor(_DevArray(buf(which), shape, ts), device=dev)
        self.f_off_loc = wrap(0, (self.n_loc, self.m), "<f8")
        self.f_gather = wrap(1, (world * self.n_loc, self.m), "<f8")
        self.best_key = wrap(2, (self.r,), "<i8")
        self.first_row = wrap(3, (self.r,), "<i4")
        self.best_row = wrap(4, (self.r,), "<i4")
        self.free_slot = wrap(5, (self.n_loc,), "<i4")
        self.free_all = wrap(6, (world * self.n_loc,), "<i4")
        self.pool_ptr = int(buf(7))
        self._torch = torch
        self._direct = direct_peers
        # every stage runs on the library's stream: collectives issued with it as the current stream are ordered
        # against the stages by NCCL's own stream events, without device-wide synchronisation
        self.stream = torch.cuda.ExternalStream(int(self._L.temo_b200_shard_stream(self._h)), device=dev)
        self.k1_events = None  # list: collect (start, end) CUDA events of every K1 launch

    def _chk(self, rc):
        if rc:
            msg = self._L.temo_b200_shard_last_error().decode(errors="replace")
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def _info(self):
        info = np.zeros(8, dtype=np.uint64)
        self._chk(self._L.temo_b200_shard_info(self._h, info.ctypes.data_as(u64p)))
        return info

    def launches(self) -> int:
        """Kernels and copies this shard has enqueued so far (counted where they are launched, csrc/shard.cu)."""
        return int(self._info()[7])

    def state(self) -> dict:
        st = np.zeros(5, dtype=np.uint64)
        self._chk(self._L.temo_b200_shard_state(self._h, st.ctypes.data_as(u64p)))
        return dict(P=int(st[0]), counter=int(st[1]), t=int(st[2]), lo=int(st[3]), hi=int(st[4]))

    def sync(self):
        self._torch.cuda.synchronize()

    def on_stream(self):
        """Context manager: torch ops (collectives) issued inside use the shard's stream as the current stream."""
        return self._torch.cuda.stream(self.stream)

    def connect_peers(self, comm) -> None:
        """Maps every peer's pool into this process (world > 1): the IPC handles travel through the communicator."""
        if self.world == 1:
            return
        if self._direct:  # several shards of one process: the pools are plain pointers
            ptrs = comm.all_gather_bytes(self.pool_ptr)
            arr = (C.c_void_p * self.world)(*[C.c_void_p(int(p)) for p in ptrs])
            self._chk(self._L.temo_b200_shard_set_peer_pointers(self._h, arr))
            return
        mine = (C.c_ubyte * 64)()
        self._chk(self._L.temo_b200_shard_ipc_handle(self._h, mine))
        handles = comm.all_gather_bytes(bytes(mine))
        blob = (C.c_ubyte * (64 * self.world)).from_buffer_copy(b"".join(handles))
        self._chk(self._L.temo_b200_shard_open_peers(self._h, blob))

    def begin(self):
        self._chk(self._L.temo_b200_shard_begin(self._h))

    def reproduce(self):
        ev = None
        if self.k1_events is not None:  # device time of the K1 launches (bench): events on the shard's stream
            ev = (self._torch.cuda.Event(enable_timing=True), self._torch.cuda.Event(enable_timing=True))
            ev[0].record(self.stream)
        self._chk(self._L.temo_b200_shard_reproduce(self._h))
        if ev is not None:
            ev[1].record(self.stream)
            self.k1_events.append(ev)

    def place_initial_f(self):
        self._chk(self._L.temo_b200_shard_place_initial_f(self._h))

    def select_local(self):
        self._chk(self._L.temo_b200_shard_select_local(self._h))

    def select_rows(self):
        self._chk(self._L.temo_b200_shard_select_rows(self._h))

    def finish(self) -> int:
        cnt = u64(0)
        self._chk(self._L.temo_b200_shard_finish(self._h, C.byref(cnt)))
        return int(cnt.value)

    def download(self) -> dict:
        st = self.state()
        P = st["P"]
        owner, slot = np.empty(P, dtype=np.uint32), np.empty(P, dtype=np.uint32)
        rows = u64(0)
        idx = np.empty(P, dtype=np.uint64)
        x = np.empty((P, self.d))
        f = np.empty((P, self.m))
        v, gamma = np.empty((self.r, self.m)), np.empty(self.r)
        u32p = C.POINTER(C.c_uint32)
        self._chk(self._L.temo_b200_shard_download(self._h, owner.ctypes.data_as(u32p), slot.ctypes.data_as(u32p), C.byref(rows),
                                                   idx.ctypes.data_as(u64p), x.ctypes.data_as(_lib.f64p), f.ctypes.data_as(_lib.f64p),
                                                   v.ctypes.data_as(_lib.f64p), gamma.ctypes.data_as(_lib.f64p)))
        k = int(rows.value)
        return dict(owner=owner, slot=slot, idx=idx[:k].astype(np.int64), x=x[:k].copy(), f=f, v=v, gamma=gamma, **st)

    def close(self):
        if self._h:
            self._L.temo_b200_shard_destroy(self._h)
            self._h = C.c_void_p()


# ------------------------------------------------------------------------------------ orchestrator
class ShardedRvea:
    """The generation loop over `world` shards. `shard` provides the stage functions and buffers
    (GpuShard, or a CPU stand-in in the tests), `comm` the collectives. All loop state (survivor tables,
    draw counter, generation) lives in the shard; nothing here is O(n) work."""

    def __init__(self, cfg: RunConfig, comm, shard):
        self.cfg, self.comm, self.shard = cfg, comm, shard
        self.rank, self.world = comm.rank, comm.world
        self.n = cfg.pop
        if self.n % (2 * self.world):
            raise ValueError("sharded run: population must be divisible by 2 * world size")
        self.d, self.m, self.r = shard.d, shard.m, shard.r
        self.n_loc = self.n // self.world
        self.timers = {}
        shard.connect_peers(comm)
        # on the shard's stream like every stage: the collective's result is only ordered against the stream it was
        # issued on, and place_initial_f reads f_gather on the library's (non-blocking) stream
        with shard.on_stream():
            comm.all_gather(shard.f_gather, shard.f_off_loc)
            shard.place_initial_f()
        shard.sync()
        comm.barrier()  # every pool holds its initial block before anybody's first K1 reads it

    @property
    def P(self):
        return self.shard.state()["P"]

    @property
    def counter(self):
        return self.shard.state()["counter"]

    def _tick(self, name, t0):
        self.timers[name] = self.timers.get(name, 0.0) + (time.perf_counter() - t0)

    def step(self) -> int:
        comm, sh = self.comm, self.shard
        t0 = time.perf_counter()
        with sh.on_stream():
            sh.begin()
            sh.reproduce()
            comm.all_gather(sh.f_gather, sh.f_off_loc)
            comm.all_gather(sh.free_all, sh.free_slot)
            sh.select_local()
            comm.all_reduce_min(sh.best_key)
            comm.all_reduce_min(sh.first_row)
            sh.select_rows()
            comm.all_reduce_min(sh.best_row)
            self._tick("enqueue", t0)
            t0 = time.perf_counter()
            cnt = sh.finish()
            self._tick("finish (incl. the wait for the device)", t0)
        return cnt


# ------------------------------------------------------------------------------------ bench entry (N > 1)
def bench_main(args, metric, workload_config, measured_peaks, ClockSampler):
    """bench.py --gpus N (N > 1; also N = 1 with TEMO_FORCE_DIST=1), launched by torchrun.
    weak scaling: the global run has N * args.pop rows (N shards of args.pop rows); strong: args.pop rows in total."""
    import torch
    import torch.distributed as dist
    from . import api as tb

    rank, world, local = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    tb.init(local)
    use_nccl = world > 1 or os.environ.get("TEMO_FORCE_DIST") == "nccl"  # "nccl": the collectives of a world of 1 through NCCL
    if use_nccl:
        if "MASTER_ADDR" not in os.environ:  # not under torchrun: a single-rank rendezvous on the loopback
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = TorchComm()
    else:
        comm = LocalComm()
    strong = args.scaling == "strong"
    pop = args.pop if strong else args.pop * world
    K, W = args.steps, args.warmup
    cfg = RunConfig(problem=args.problem, pop=pop, dim=args.dim, obj=args.obj, generations=max(100, W + K + 2), seed=args.seed,
                    fuse_eval=False if args.no_fuse else None)
    shard = GpuShard(cfg, rank, world)
    run = ShardedRvea(cfg, comm, shard)
    for _ in range(W):
        run.step()
    run.timers.clear()
    shard.k1_events = []
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    launches0, calls0 = shard.launches(), comm.calls
    comm.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(shard.stream)
    t0 = time.perf_counter()
    for _ in range(K):
        pop_size = run.step()
    stop.record(shard.stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    comm.barrier()
    wall = comm.all_reduce_max_scalar(max(wall, start.elapsed_time(stop) * 1e-3))  # max over ranks
    clocks = sampler.stop() if rank == 0 else None
    if rank == 0:
        peak, peak_src = measured_peaks()
        nd = float(run.n_loc) * run.d
        rep_ms = sum(a.elapsed_time(b) for a, b in shard.k1_events) / K  # K1 launch of one step (CUDA events)
        args_cfg = workload_config(args, None)
        shards = f"{world} shards of {run.n_loc} rows"
        args_cfg.update({"workload": f"RVEA/{args.problem} m={args.obj} d={args.dim} pop={pop} ({shards})", "pop": pop,
                         "ref_vectors": run.r, "survivors_last": int(pop_size), "scaling_mode": args.scaling,
                         "parents": "NVLink peer loads inside K1 (CUDA IPC mapped pools); no row exchange collective"})
        gens_per_s = K / wall  # generations of the GLOBAL population per second
        # weak scaling: per-GPU work is fixed, the job advances `world` shards of args.pop rows per step: the aggregate in
        # the metric's unit (generations of one args.pop-row population per second) is world * gens_per_s
        value = gens_per_s if strong else world * gens_per_s
        if not strong:
            args_cfg["unit_note"] = (f"value = {world} x {gens_per_s:.2f} global generations/s: every step advances {world} shards of "
                                     f"{args.pop} rows (one RVEA run of {pop} rows)")
        line = {
            "metric": metric, "value": value, "unit": "generations/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": wall / K * 1e3, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": args_cfg,
            "global_generations_per_s": gens_per_s, "rows_per_s": K * float(pop) / wall,
            # per step and rank: the mating permutation goes up, the survivor count and status words come back
            "e2e": {"value": value, "unit": "generations/s", "h2d_bytes_per_step": 4 * pop, "d2h_bytes_per_step": 12},
            "gpu_launches": int(shard.launches() - launches0),
            "collectives": int(comm.calls - calls0),
            "roofline": {"bound": "hbm", "kernel": "reproduce_pairs_kernel (rank 0, CUDA events around the K1 launch of every step; remote "
                                                   "parents arrive over NVLink inside it)",
                         "achieved": 16.0 * nd / (rep_ms * 1e-3) / 1e9 if rep_ms else None,
                         "peak": peak, "unit": "GB/s", "frac": (16.0 * nd / (rep_ms * 1e-3) / 1e9 / peak) if rep_ms else None, "traffic": None,
                         "peak_source": peak_src},
            "stages_ms": {**{k: v / K * 1e3 for k, v in run.timers.items()}, "reproduce_device": rep_ms},
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    shard.close()
    if use_nccl:
        dist.destroy_process_group()
