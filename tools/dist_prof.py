import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import paper_2404_01159_b200 as tb
from paper_2404_01159_b200 import dist as td
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29533"); os.environ.setdefault("RANK","0"); os.environ.setdefault("WORLD_SIZE","1")
torch.cuda.set_device(0); tb.init(0)
dist.init_process_group("nccl", device_id=torch.device("cuda",0))
comm = td.TorchComm()
cfg = tb.RunConfig(problem="dtlz2", pop=1<<17, dim=5000, obj=3, generations=100, seed=42)
shard = td.GpuShard(cfg, 0, 1)
run = td.ShardedRvea(cfg, comm, shard)
# monkeypatch fine timers
T = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
    setattr(obj, name, g)
for n in ["pack","reproduce","place_f","select_local","select_rows","select_finish","commit","free_slots_host"]: wrap(shard, n)
for n in ["all_to_all_rows","all_gather","all_reduce_min"]: wrap(comm, n)
import paper_2404_01159_b200.dist as D
sp = D.shard_plan
def sp2(*a, **k):
    t0=time.perf_counter(); r=sp(*a, **k); T["shard_plan"]=T.get("shard_plan",0)+time.perf_counter()-t0; return r
D.shard_plan = sp2
for _ in range(3): run.step()
T.clear(); run.timers.clear()
K=10
t0=time.perf_counter()
for _ in range(K): run.step()
torch.cuda.synchronize()
print("step ms", (time.perf_counter()-t0)/K*1e3)
for k,v in sorted(T.items(), key=lambda kv:-kv[1]): print(f"{k:18s} {v/K*1e3:7.3f} ms")
print({k: round(v/K*1e3,3) for k,v in run.timers.items()})
