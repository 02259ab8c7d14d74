"""Multi-GPU parity: the distributed round loop on N GPUs (one rank per GPU)
with the peer-memory and the NCCL transports == the oracle's run_parallel.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/dist_parity.py
Prints one line per case on rank 0 and exits non-zero on a mismatch."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import torch.distributed as dist

import paper_2601_01787_b200 as pm
from oracle import oracle as orc
from paper_2601_01787_b200 import dist as pdist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    bad = 0
    cases = [((48, 40, 16 * world), (1, 1, world), 3, 1e-2), ((16 * world, 30, 20), (world, 1, 1), 4, 1e-2)]
    if world >= 4:
        cases.append(((40, 36, 28), pdist.block_grid(world), 5, 1e-2))
    for dims, grid, seed, rel in cases:
        f = orc.perlin(dims, seed)
        xi = orc.relative_to_absolute(f, rel)
        fh = orc.quantize(f, xi)
        cfg = pm.CorrectionConfig(xi_abs=xi)
        blocks = pm.decompose(dims, grid).blocks
        b = blocks[rank]
        nx, ny, nz = dims
        sl = b.ext_slices_zyx()
        fe = torch.from_numpy(np.ascontiguousarray(f.reshape(nz, ny, nx)[sl]).reshape(-1)).to(dev)
        he = torch.from_numpy(np.ascontiguousarray(fh.reshape(nz, ny, nx)[sl]).reshape(-1)).to(dev)
        for lockstep in (False, True):
            ref_g, ref = (orc.run_parallel(dims, f, fh, xi, grid, lockstep) if rank == 0 else (None, None))
            for kind in ("peer", "collective", "devloop"):
                eng = pdist.DeviceEngine(b, dims, fe, he, cfg)
                eng.prepare()
                os.environ["PMSZ_DEVLOOP"] = "1" if kind == "devloop" else "0"
                if kind in ("peer", "devloop"):
                    tp = pdist.PeerTransport(eng, blocks, rank)
                    tp.connect()
                else:
                    tp = pdist.CollectiveTransport(eng, blocks, rank)
                st = pdist.run_distributed(eng, blocks, grid, rank, lockstep, cfg.max_outer_iterations, transport=tp)
                sp = eng.spec
                ed = sp.dims
                core = eng.g.cpu().numpy().reshape(ed[2], ed[1], ed[0])[
                    sp.core_lo[2]:sp.core_hi[2], sp.core_lo[1]:sp.core_hi[1], sp.core_lo[0]:sp.core_hi[0]].copy()
                parts = [None] * world
                dist.all_gather_object(parts, (core, eng.block_stats()))
                if rank == 0:
                    g = np.empty((nz, ny, nx))
                    for bb, (c, _) in zip(blocks, parts):
                        g[bb.core_slices_zyx()] = c
                    ok = (np.array_equal(g.reshape(-1), ref_g) and (st.rounds, st.syncs) == (ref["rounds"], ref["syncs"])
                          and tuple(st.edits_per_round) == tuple(ref["edits_per_iteration"])
                          and tuple(p[1][1] for p in parts) == tuple(ref["per_block_edit_totals"]))
                    bad += not ok
                    print(f"{'OK ' if ok else 'BAD'} dims={dims} grid={grid} {'lockstep' if lockstep else 'relaxed'} "
                          f"{kind} rounds={st.rounds} syncs={st.syncs}", flush=True)
    bad += golden_256(rank, world, dev)
    t = torch.tensor([bad], device=dev)
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    return int(t.item())


def golden_256(rank, world, dev) -> int:
    """Benchmark-scale multi-GPU parity: Perlin 256^3 (seed 0, f32, rel 1e-4,
    quantizer) on z-slabs (1, 1, world), relaxed, the C round loop over NVLink
    -- the corrected field and the whole ParallelStats against the
    reference's own run_parallel (tests/golden/golden_large.json, c256)."""
    import hashlib
    import json
    from paper_2601_01787_b200 import inputs as gen
    ref = json.loads((Path(__file__).resolve().parent.parent / "tests" / "golden" / "golden_large.json").read_text())
    case = next((c for c in ref["c256"]["parallel"] if c["grid"] == [1, 1, world] and c["strategy"] == "relaxed"), None)
    if case is None:
        return 0
    dims = (256, 256, 256)
    blocks = pm.decompose(dims, (1, 1, world)).blocks
    b = blocks[rank]
    spec = gen.NoiseSpec(dims, 0)
    f32 = gen.perlin_device(spec, lo=b.ext_start, ext=b.ext_dims, f32=True, device=dev)
    lo, hi = gen.minmax_device(f32)
    mm = torch.tensor([-lo, hi], dtype=torch.float64, device=dev)
    dist.all_reduce(mm, op=dist.ReduceOp.MAX)
    glo, ghi = -float(mm[0].item()), float(mm[1].item())
    xi = gen.relative_to_absolute_range(glo, ghi, 1e-4)
    fh = gen.quantize_device(f32, xi, glo, ghi)
    cfg = pm.CorrectionConfig(xi_abs=xi)
    eng = pdist.DeviceEngine(b, dims, f32, fh, cfg)
    eng.prepare()
    os.environ["PMSZ_DEVLOOP"] = "1"
    tp = pdist.make_transport(eng, blocks, rank)
    st = pdist.run_distributed(eng, blocks, (1, 1, world), rank, False, cfg.max_outer_iterations, transport=tp)
    sp = eng.spec
    nx, ny = dims[0], dims[1]
    core = eng.g[sp.core_lo[2] * nx * ny: sp.core_hi[2] * nx * ny].contiguous()
    parts = [torch.empty_like(core) for _ in range(world)]   # equal slabs: 256 % world == 0
    dist.all_gather(parts, core)
    stats = [None] * world
    dist.all_gather_object(stats, eng.block_stats())
    if rank != 0:
        return 0
    g = torch.cat(parts).cpu().numpy()
    d = case["stats"]
    ok = (hashlib.sha256(g.tobytes()).hexdigest() == case["corrected_sha256"]
          and (st.rounds, st.syncs) == (d["rounds"], d["syncs"])
          and list(st.edits_per_round) == case["edits_per_iteration"]
          and [s[0] for s in stats] == d["per_block_iterations"]
          and [s[1] for s in stats] == d["per_block_edit_totals"]
          and [s[2] for s in stats] == d["per_block_max_vertex_edits"])
    print(f"{'OK ' if ok else 'BAD'} dims={dims} grid=(1, 1, {world}) relaxed devloop vs reference run_parallel "
          f"(golden_large c256) rounds={st.rounds} syncs={st.syncs}", flush=True)
    return int(not ok)


if __name__ == "__main__":
    sys.exit(1 if main() else 0)
