"""Row-block sharding on the device, emulated on one GPU by running the ranks one after another
(never concurrently): shards -> gathered tree -> per-rank row_range multiply.  The union of the
per-rank products must be bit-identical to the single-GPU product, for any number of ranks."""

import numpy as np
import pytest
import torch

from paper_1203_1692_b200 import inputs, parallel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_row_blocks_reproduce_single_gpu_product(world):
    import paper_1203_1692_b200 as P
    n, tau = 1024, 1e-6
    a = inputs.exponential_decay(n, 0.9, seed=0)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau)
    c_ref, plan_ref, k_ref = P.multiply(qa, qa, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = n // 16
    # what the ranks would hold, and what the all-gather would deliver (rank order)
    shards = [parallel.shard_from_dense_rows(a[r0 * 16:r1 * 16], r0) for r0, r1 in parallel.even_row_split(nrows, world)]
    gathered = parallel.PackedShard(torch.cat([s.keys for s in shards]), torch.cat([s.records for s in shards]),
                                    torch.cat([s.leaf_sq for s in shards]))
    full = parallel.tree_from_shard(n, n, gathered)
    # the gathered tree is the same matrix with the same norms
    assert np.array_equal(full.to_dense().data, a)
    for t in range(qa.depth + 1):
        assert np.array_equal(full.level_norms(t), qa.level_norms(t))
    plan = P.build_plan(full, full, tau)
    assert len(plan) == len(plan_ref)
    counts = parallel.row_task_counts(plan, plan.depth).cpu().numpy()
    assert counts.sum() == len(plan)
    assert np.array_equal(counts, np.bincount(plan.ikj()[:, 0], minlength=counts.size))
    split = parallel.balanced_row_split(counts[:nrows], world)
    got = np.zeros_like(dense_ref)
    total_tasks = total_p4 = 0
    for r0, r1 in split:
        c, p, k = P.numeric.multiply_async(full, full, cfg, None, row_range=(r0, r1))
        d = c.to_dense().data
        assert not d[:r0 * 16].any() and not d[r1 * 16:].any()
        got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        total_tasks += len(p)
        total_p4 += k.products4
        rows = p.ikj()[:, 0]
        assert rows.size == 0 or (rows.min() >= r0 and rows.max() < r1)
    assert total_tasks == len(plan_ref) and total_p4 == k_ref.products4
    assert np.array_equal(got, dense_ref)
    loads = np.array([counts[r0:r1].sum() for r0, r1 in split])
    assert loads.max() <= 1.35 * loads.mean()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_local_rows_of_a_times_gathered_b(world):
    """parallel.multiply_sharded's data flow without the collective: every rank multiplies a tree of
    its own rows of A by B rebuilt from the gathered buffer (fixed stride per rank, HOLE keys in
    the unused slots, no transposed copies) and gets exactly its rows of the single-GPU product."""
    import paper_1203_1692_b200 as P
    n, tau = 1000, 1e-6                       # ragged: 62.5 leaf rows
    a = inputs.exponential_decay(n, 0.9, seed=2)
    b = inputs.exponential_decay(n, 0.93, seed=5)
    qa, qb = P.QuadtreeMatrix.from_dense(a), P.QuadtreeMatrix.from_dense(b)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    c_ref, plan_ref, k_ref = P.multiply(qa, qb, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = -(-n // 16)
    split = parallel.even_row_split(nrows, world)
    b_shards = [parallel.shard_of_tree(qb, r0, r1) for r0, r1 in split]
    cap = max(s.n for s in b_shards)
    dev = b_shards[0].keys.device
    keys = torch.full((world * cap,), parallel.HOLE, dtype=torch.int32, device=dev)
    recs = torch.full((world * cap, 272), float("nan"), dtype=torch.float32, device=dev)   # garbage must never be read
    sq = torch.zeros((world * cap,), dtype=torch.float64, device=dev)
    for r, s in enumerate(b_shards):
        keys[r * cap:r * cap + s.n] = s.keys
        recs[r * cap:r * cap + s.n] = s.records
        sq[r * cap:r * cap + s.n] = s.leaf_sq
    b_full = parallel.tree_from_shard(n, n, parallel.PackedShard(keys, recs, sq), transposed=False)
    assert np.array_equal(b_full.to_dense().data, b)
    bk, bv, bs = b_full.packed_leaves()
    rk, rv, rs = qb.packed_leaves()
    assert np.array_equal(bk, rk) and np.array_equal(bv, rv) and np.array_equal(bs, rs)
    got = np.zeros_like(dense_ref)
    tasks = p4 = 0
    for r0, r1 in split:
        a_local = parallel.tree_from_shard(n, n, parallel.shard_of_tree(qa, r0, r1))
        c, p, k = P.numeric.multiply_async(a_local, b_full, cfg, None)
        d = c.to_dense().data
        assert not d[:r0 * 16].any() and not d[r1 * 16:].any()
        got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        tasks += len(p)
        p4 += k.products4
    assert tasks == len(plan_ref) and p4 == k_ref.products4
    assert np.array_equal(got, dense_ref)
    # a right-hand-only tree still works on the left: the transposed copies are made on first use
    c2, _, _ = P.multiply(b_full, qa, P.MultiplyConfig(tau=tau, exact=True))
    c3, _, _ = P.multiply(qb, qa, P.MultiplyConfig(tau=tau, exact=True))
    assert np.array_equal(c2.to_dense().data, c3.to_dense().data)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_band_limited_exchange_gives_the_same_rows(world):
    """exchange="needed": a rank multiplies its rows of A by ONLY the leaf rows of B its columns
    reach (what parallel.exchange_needed_rows delivers, pieces in owner order).  Rows of C must be
    bit-identical to the single-GPU product, and for a banded matrix most of B is never fetched."""
    import paper_1203_1692_b200 as P
    n, tau = 2048, 1e-6
    a = inputs.exponential_decay(n, 0.5, seed=0)            # narrow band: entries underflow ~150 columns out
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    c_ref, plan_ref, k_ref = P.multiply(qa, qa, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = n // 16
    split = parallel.even_row_split(nrows, world)
    shards = [parallel.shard_of_tree(qa, r0, r1) for r0, r1 in split]
    got = np.zeros_like(dense_ref)
    tasks = fetched = 0
    for rank, (r0, r1) in enumerate(split):
        need = parallel.needed_rows(shards[rank], nrows)
        rows_of = [parallel._squeeze16(s.keys.to(torch.int64) >> 1) for s in shards]
        pieces = [torch.nonzero(need[rows_of[src]]).flatten() for src in range(world)]
        part = parallel.PackedShard(torch.cat([shards[s].keys[pieces[s]] for s in range(world)]),
                                    torch.cat([shards[s].records[pieces[s]] for s in range(world)]),
                                    torch.cat([shards[s].leaf_sq[pieces[s]] for s in range(world)]))
        fetched += part.n - int(pieces[rank].numel())
        b_part = parallel.tree_from_shard(n, n, part, transposed=False)
        a_local = parallel.tree_from_shard(n, n, shards[rank])
        c, p, k = P.numeric.multiply_async(a_local, b_part, cfg, None)
        d = c.to_dense().data
        got[r0 * 16:r1 * 16] = d[r0 * 16:r1 * 16]
        assert not d[:r0 * 16].any() and not d[r1 * 16:].any()
        tasks += len(p)
    assert tasks == len(plan_ref)
    assert np.array_equal(got, dense_ref)
    if world == 8:
        assert fetched < 0.3 * (world - 1) * qa.nleaf          # an all-gather would move (world-1) * nleaf


@pytest.mark.parametrize("world", [2, 4])
def test_interior_rows_first_gives_the_same_rows(world):
    """ShardedMultiply's overlap, emulated rank by rank without the collective: the interior rows of a
    rank's block (whose tasks only touch the rank's own rows of B) are multiplied against a tree that
    holds ONLY those own rows -- what is available before the exchange has finished -- and the rows
    above and below against B limited to what the band-limited exchange delivers.  The rows of C must be
    bit-identical to the single-GPU product."""
    import paper_1203_1692_b200 as P
    n, tau = 2048, 1e-6
    a = inputs.exponential_decay(n, 0.8, seed=1)
    qa = P.QuadtreeMatrix.from_dense(a)
    cfg = P.MultiplyConfig(tau=tau, exact=True)
    c_ref, plan_ref, k_ref = P.multiply(qa, qa, cfg)
    dense_ref = c_ref.to_dense().data
    nrows = n // 16
    split = parallel.even_row_split(nrows, world)
    shards = [parallel.shard_of_tree(qa, r0, r1) for r0, r1 in split]
    whole = parallel.shard_of_tree(qa, 0, nrows)
    rowmax = parallel.row_max_norms(whole, nrows)
    got = np.zeros_like(dense_ref)
    tasks = 0
    for rank, (r0, r1) in enumerate(split):
        mine = shards[rank]
        reach = parallel.reaching_leaves(mine, rowmax, tau)
        i0, i1 = parallel.interior_rows(mine, (r0, r1), split[rank], reach)
        assert i1 > i0
        need = parallel.needed_rows(mine, nrows, reach)
        rows_of = [parallel._squeeze16(s.keys.to(torch.int64) >> 1) for s in shards]
        pieces = [torch.nonzero(need[rows_of[src]]).flatten() for src in range(world)]
        part = parallel.PackedShard(torch.cat([shards[s].keys[pieces[s]] for s in range(world)]),
                                    torch.cat([shards[s].records[pieces[s]] for s in range(world)]),
                                    torch.cat([shards[s].leaf_sq[pieces[s]] for s in range(world)]))
        a_local = parallel.tree_from_shard(n, n, mine)
        b_own = parallel.tree_from_shard(n, n, mine, transposed=False)
        b_part = parallel.tree_from_shard(n, n, part, transposed=False)
        for (lo, hi), b in (((i0, i1), b_own), ((r0, i0), b_part), ((i1, r1), b_part)):
            if hi <= lo:
                continue
            c, p, k = P.numeric.multiply_async(a_local, b, cfg, None, row_range=(lo, hi))
            d = c.to_dense().data
            assert not d[:lo * 16].any() and not d[hi * 16:].any()
            got[lo * 16:hi * 16] = d[lo * 16:hi * 16]
            tasks += len(p)
    assert tasks == len(plan_ref)
    assert np.array_equal(got, dense_ref)


def test_sharded_multiply_under_a_one_rank_nccl_group():
    """The real entry points (ShardedMultiply, multiply_sharded) under torch.distributed with the NCCL
    backend and a single rank: the product must be the plain multiply's, bit for bit."""
    import os
    import socket
    import torch.distributed as dist
    import paper_1203_1692_b200 as P
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        n, tau = 1024, 1e-6
        a = inputs.exponential_decay(n, 0.9, seed=0)
        qa = P.QuadtreeMatrix.from_dense(a)
        cfg = P.MultiplyConfig(tau=tau, exact=True)
        want = P.multiply(qa, qa, cfg)[0].to_dense().data
        nrows = n // 16
        mine = parallel.shard_of_tree(qa, 0, nrows)
        for exchange in ("all", "needed", "auto"):
            sm = parallel.ShardedMultiply(mine, None, (n, n), (n, n), cfg, splits=[(0, nrows)], exchange=exchange)
            for _ in range(2):
                res = sm.run()
                assert len(res) == 1 and res[0][0] == (0, nrows)
                assert np.array_equal(res[0][1].to_dense().data, want)
        c, plan, k = parallel.multiply_sharded(mine, None, (n, n), (n, n), cfg, exchange="needed", splits=[(0, nrows)])
        assert np.array_equal(c.to_dense().data, want)
        c, plan, k = parallel.multiply_sharded(mine, None, (n, n), (n, n), cfg, exchange="all")
        assert np.array_equal(c.to_dense().data, want)
        # alpha == 0 gives an empty product, beta != 0 is refused (only C = alpha A B is sharded)
        c0, _, _ = parallel.multiply_sharded(mine, None, (n, n), (n, n), P.MultiplyConfig(tau=tau, alpha=0.0), exchange="all")
        assert c0.nleaf == 0
        with pytest.raises(ValueError):
            parallel.multiply_sharded(mine, None, (n, n), (n, n), P.MultiplyConfig(tau=tau, beta=1.0), exchange="all")
    finally:
        dist.destroy_process_group()


def test_c_abi_allgather_with_a_raw_nccl_communicator():
    """spamm_exchange_allgather takes the caller's ncclComm_t.  With a one-rank
    communicator made straight from NCCL (no torch.distributed) the gathered buffers must equal the
    rank's padded shard, and the tree indexed on them must be the original matrix."""
    import ctypes as C
    import glob
    import os
    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import _lib
    import nvidia.nccl
    path = glob.glob(os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so*"))[0]
    nccl = C.CDLL(path, mode=C.RTLD_GLOBAL)

    class UniqueId(C.Structure):
        _fields_ = [("internal", C.c_char * 128)]

    uid, comm = UniqueId(), C.c_void_p()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    try:
        n = 512
        a = inputs.exponential_decay(n, 0.9, seed=7)
        qa = P.QuadtreeMatrix.from_dense(a)
        mine = parallel.shard_of_tree(qa, 0, n // 16)
        cap = mine.n + 5                                   # a few unused slots, as when shards differ in size
        dev = mine.keys.device
        keys = torch.full((cap,), parallel.HOLE, dtype=torch.int32, device=dev)
        recs = torch.zeros((cap, 272), dtype=torch.float32, device=dev)
        sq = torch.zeros((cap,), dtype=torch.float64, device=dev)
        keys[:mine.n], recs[:mine.n], sq[:mine.n] = mine.keys, mine.records, mine.leaf_sq
        out = parallel.PackedShard(torch.empty_like(keys), torch.empty_like(recs), torch.empty_like(sq))
        st = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.lib().spamm_exchange_allgather(comm, keys.data_ptr(), recs.data_ptr(), sq.data_ptr(), cap,
                                                       out.keys.data_ptr(), out.records.data_ptr(), out.leaf_sq.data_ptr(),
                                                       st), "exchange_allgather")
        torch.cuda.synchronize()
        assert torch.equal(out.keys, keys) and torch.equal(out.records, recs) and torch.equal(out.leaf_sq, sq)
        b_full = parallel.tree_from_shard(n, n, out, transposed=False)
        assert np.array_equal(b_full.to_dense().data, a)
    finally:
        nccl.ncclCommDestroy.argtypes = [C.c_void_p]
        nccl.ncclCommDestroy(comm)


def test_sharded_multiply_on_two_gpus():
    """ShardedMultiply and multiply_sharded under torchrun with one rank per GPU (NCCL over NVLink): every rank's
    rows of C equal the single-GPU product bit for bit, for both exchanges, with and without the overlap of the
    interior rows.  Skipped on a single-GPU box (the CPU suite runs the same logic with gloo, world size 2)."""
    import os
    import subprocess
    import sys
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs at least 2 GPUs")
    world = 2 if ngpu < 4 else 4
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", "29541", os.path.join(root, "tests", "sharded_child.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert f"SHARDED OK {world}" in out.stdout
