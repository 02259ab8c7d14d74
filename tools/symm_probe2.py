"""Probe the relaxed-round exchange primitives on 2+ GPUs (symmetric memory)."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
n = 512 * 512 * 2
buf = symm.empty(n + 8, dtype=torch.float64, device=dev)
h = symm.rendezvous(buf, dist.group.WORLD.group_name)
peer = (rank + 1) % world
pb = h.get_buffer(peer, (n + 8,), torch.float64)
src = torch.randn(n, dtype=torch.float64, device=dev)
loc = torch.empty(n, dtype=torch.float64, device=dev)
hin = torch.zeros(8, dtype=torch.float64, pin_memory=True)
hout = torch.zeros(8, dtype=torch.float64, pin_memory=True)
sums = [h.get_buffer(r, (n + 8,), torch.float64)[n:] for r in range(world)]


def timeit(label, fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    h.barrier(channel=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    if rank == 0:
        print(f"{label:45s} dev {e0.elapsed_time(e1) * 1e3 / reps:8.1f} us   host {(time.perf_counter() - t0) * 1e6 / reps:8.1f} us",
              flush=True)


timeit("local copy 4MB into symm buffer", lambda: buf[:n].copy_(src))
timeit("local copy 4MB plain", lambda: loc.copy_(src))
timeit("barrier", lambda: h.barrier(channel=0))
timeit("P2P read copy 4MB (peer -> local)", lambda: loc.copy_(pb[:n]))
timeit("P2P write copy 4MB (local -> peer)", lambda: pb[:n].copy_(src))
def sums_read():
    hin.numpy()[:2] = [1, 2]
    sums[rank][:2].copy_(hin[:2], non_blocking=True)
    h.barrier(channel=0)
    hout[:2].copy_(torch.stack([s[:2] for s in sums]).sum(0), non_blocking=True)
    torch.cuda.current_stream().synchronize()
timeit("sums publish+barrier+read+sync", sums_read)
def host_sync():
    torch.cuda.current_stream().synchronize()
timeit("stream sync (idle)", host_sync)
dist.barrier()
dist.destroy_process_group()
