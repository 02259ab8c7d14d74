"""Probe: torch symmetric memory between ranks (P2P over NVLink)."""
import os, time, torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
n = 512 * 512 * 2
buf = symm.empty(n, dtype=torch.float64, device=dev)
h = symm.rendezvous(buf, dist.group.WORLD.group_name)
buf.fill_(rank + 1)
h.barrier(channel=0)
peer = (rank + 1) % world
pb = h.get_buffer(peer, (n,), torch.float64)
print(rank, "peer value", float(pb[0].item()), float(pb[-1].item()), flush=True)
out = torch.empty(n, dtype=torch.float64, device=dev)
for _ in range(5):
    h.barrier(channel=0); out.copy_(pb)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    h.barrier(channel=0)
    out.copy_(pb)
e1.record()
torch.cuda.synchronize()
print(rank, "barrier+4MB peer copy us", e0.elapsed_time(e1) * 10, "host us", (time.perf_counter() - t0) * 1e4, flush=True)
# NCCL send/recv for comparison
recv = torch.empty(n, dtype=torch.float64, device=dev)
send = torch.full((n,), float(rank), dtype=torch.float64, device=dev)
for _ in range(3):
    ops = [dist.P2POp(dist.isend, send, peer), dist.P2POp(dist.irecv, recv, (rank - 1) % world)]
    for r in dist.batch_isend_irecv(ops): r.wait()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    ops = [dist.P2POp(dist.isend, send, peer), dist.P2POp(dist.irecv, recv, (rank - 1) % world)]
    for r in dist.batch_isend_irecv(ops): r.wait()
torch.cuda.synchronize()
print(rank, "nccl sendrecv 4MB us", (time.perf_counter() - t0) * 1e4, flush=True)
dist.destroy_process_group()
