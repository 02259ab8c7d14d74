"""Multi-rank host logic on CPU: the distributed round loop (dist.py) with 2
gloo ranks and the oracle engine reproduces the oracle's single-process
run_parallel (pinned to the reference) bit for bit, stats included."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, grid, seed, rel, lockstep, out):
    import paper_2601_01787_b200 as pm
    from oracle.dist_engine import OracleEngine
    from paper_2601_01787_b200 import dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f = orc.perlin(dims, seed)
        xi = orc.relative_to_absolute(f, rel)
        fh = orc.quantize(f, xi)
        cfg = pm.CorrectionConfig(xi_abs=xi)
        blocks = pm.decompose(dims, grid).blocks
        spec = pm.block_domain(blocks[rank], dims)
        eng = OracleEngine(blocks[rank], spec, dims, f, fh, xi, cfg.tau, cfg.max_outer_iterations)
        st = pdist.run_distributed(eng, blocks, grid, rank, lockstep, cfg.max_outer_iterations)
        cores = [None] * world
        dist.all_gather_object(cores, (eng.core_values(spec).copy(), st.iterations, st.edit_total,
                                       st.max_vertex_edits))
        if rank == 0:
            out.put((st.rounds, st.syncs, st.edits_per_round, cores))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,grid,seed,rel,lockstep", [
    ((16, 16, 24), (1, 1, 2), 9, 1e-2, False),
    ((16, 16, 24), (1, 1, 2), 9, 1e-2, True),
    ((20, 18, 12), (2, 1, 1), 4, 1e-1, False),
    ((12, 20, 10), (1, 2, 1), 5, 1e-1, True),
])
def test_two_rank_round_loop_matches_oracle_run_parallel(dims, grid, seed, rel, lockstep):
    import paper_2601_01787_b200 as pm
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, grid, seed, rel, lockstep, out)) for r in range(2)]
    for p in procs:
        p.start()
    rounds, syncs, totals, cores = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = orc.perlin(dims, seed)
    xi = orc.relative_to_absolute(f, rel)
    ref_g, ref = orc.run_parallel(dims, f, orc.quantize(f, xi), xi, grid, lockstep)
    assert (rounds, syncs) == (ref["rounds"], ref["syncs"])
    assert tuple(totals) == ref["edits_per_iteration"]
    assert tuple(c[1] for c in cores) == ref["per_block_iterations"]
    assert tuple(c[2] for c in cores) == ref["per_block_edit_totals"]
    assert tuple(c[3] for c in cores) == ref["per_block_max_vertex_edits"]
    nx, ny, nz = dims
    g = np.empty((nz, ny, nx))
    for b, (vals, *_rest) in zip(pm.decompose(dims, grid).blocks, cores):
        g[b.core_slices_zyx()] = vals
    assert np.array_equal(g.reshape(-1), ref_g)


def test_exchange_topology():
    import paper_2601_01787_b200 as pm
    from paper_2601_01787_b200.dist import exchanges
    blocks = pm.decompose((8, 8, 32), (1, 1, 4)).blocks
    xs = exchanges(blocks, 1)
    assert [x.peer for x in xs] == [0, 2]
    # two planes: ghost + first core layer on each side
    assert xs[0].lo == (0, 0, 0) and xs[0].hi == (8, 8, 2)
    assert xs[1].hi[2] - xs[1].lo[2] == 2
    # 2x2x2 blocks: all 7 others overlap (full ext overlaps incl. mixed-sign corners, H12)
    b8 = pm.decompose((12, 12, 12), (2, 2, 2)).blocks
    assert len(exchanges(b8, 0)) == 7
