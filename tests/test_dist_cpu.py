"""Multi-GPU partition and exchange logic on CPU.

paper_1209_5421_b200/partition.py states the partition rules of
setup_device_dist (csrc/setup.cu); tests/test_gpu_dist.py pins it to the CUDA
library (part_dofs).  Here two gloo ranks run the exchange schedule of the
finest level -- ghost requests / replies, ghost refresh before every colour
pass, all-reduced inner products -- on a numpy restatement of the finest
colour pass, and must reproduce the one-process result bitwise."""
import os
import socket

import numpy as np
import pytest

from paper_1209_5421_b200 import partition as pt
from paper_1209_5421_b200 import problems


def _prob():
    return problems.jittered_p1(129)   # N = 16,641, L = 7: 128 x 128 level-L cells


@pytest.mark.parametrize("parts", [1, 2, 4, 8])
def test_partition_covers_and_ghosts_are_symmetric(parts):
    s = _prob()
    P = pt.Partition(s.A, s.coords, parts)
    owned = [P.owned_dofs(r) for r in range(parts)]
    allids = np.concatenate(owned)
    assert np.array_equal(np.sort(allids), np.arange(s.A.n_rows))
    counts = np.array([P.ghost_counts(r) for r in range(parts)])
    assert np.all(np.diag(counts) == 0)
    # A is symmetric: q needs something from r iff r needs something from q
    assert np.array_equal(counts > 0, (counts > 0).T)
    for r in range(parts):
        g = P.ghosts(r)
        assert np.all(P.owner[g] != r)
        assert np.all(np.diff(P.owner[g]) >= 0)   # grouped by owner


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_ring_boxes_pair_up(parts):
    for w in (32, 64, 256):
        for r in range(parts):
            send, _ = pt.ring_boxes(w, parts, r)
            for q, box in send.items():
                _, recv_q = pt.ring_boxes(w, parts, q)
                assert recv_q[r] == box


def test_level_plan_agglomerates_once():
    s = problems.jittered_p1(513)   # L = 9, 512 x 512 level-L cells
    # deep plan (AUX_DIST_AGG_SIDE=0): distributed while the rectangles stay tileable
    for parts, first_gathered_k in ((2, 4), (4, 4), (8, 5)):
        plan = pt.Partition(s.A, s.coords, parts).level_plan(agg_side=0)
        d = [lv["dist"] for lv in plan]
        assert d[0] and not d[-1]
        assert d == sorted(d, reverse=True)            # distributed levels come first
        k_agg = next(lv["k"] for lv in plan if not lv["dist"])
        assert k_agg == first_gathered_k
    # the library's default (agg_side 512): only level L (512 wide) stays distributed
    for parts in (2, 4, 8):
        plan = pt.Partition(s.A, s.coords, parts).level_plan(agg_side=512)
        assert [lv["dist"] for lv in plan][:2] == [True, False]


# ---------------------------------------------------------------- 2 gloo ranks

def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _colour_pass_serial(A, x, b, P, colour_rows):
    """Block-GS colour pass (smoother.hpp:162-205) with residuals taken before
    the updates (colour-clean snapshot semantics), blocks = level-L cells."""
    Ad = A
    x = x.copy()
    for cells in colour_rows:
        r = {}
        for rows in cells:
            r[tuple(rows)] = b[rows] - Ad[rows] @ x
        for rows in cells:
            blk = Ad[np.ix_(rows, rows)]
            x[rows] = x[rows] + np.linalg.solve(blk, r[tuple(rows)])
    return x


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = _prob()
        A = s.A
        import scipy.sparse as sp
        Ad = sp.csr_matrix((A.values, A.col_idx, A.row_ptr), shape=(A.n_rows, A.n_rows)).toarray()
        P = pt.Partition(A, s.coords, world)
        mine = P.owned_dofs(rank)
        ghosts = P.ghosts(rank)
        gcount = P.ghost_counts(rank)
        # request / reply: every part tells each other part how many (and which) DoFs it needs
        req_n = torch.tensor(gcount, dtype=torch.int64)
        got_n = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got_n, req_n)
        need_from_me = {qq: int(got_n[qq][rank]) for qq in range(world) if qq != rank}
        off = np.concatenate([[0], np.cumsum(gcount)])
        ops = []
        reqs = {}
        for qq in range(world):
            if qq == rank:
                continue
            if gcount[qq]:
                ops.append(dist.isend(torch.from_numpy(ghosts[off[qq]:off[qq + 1]].astype(np.int64)), qq))
            if need_from_me[qq]:
                reqs[qq] = torch.zeros(need_from_me[qq], dtype=torch.int64)
                ops.append(dist.irecv(reqs[qq], qq))
        for op in ops:
            op.wait()
        send_lists = {qq: reqs[qq].numpy() for qq in reqs}
        assert all(np.all(P.owner[v] == rank) for v in send_lists.values())

        def refresh(x_glob_view):
            """ghost refresh: send owned values each neighbour asked for, receive mine."""
            ops, bufs = [], {}
            for qq, ids in send_lists.items():
                ops.append(dist.isend(torch.from_numpy(x_glob_view[ids].copy()), qq))
            for qq in range(world):
                if qq != rank and gcount[qq]:
                    bufs[qq] = torch.zeros(int(gcount[qq]), dtype=torch.float64)
                    ops.append(dist.irecv(bufs[qq], qq))
            for op in ops:
                op.wait()
            for qq, buf in bufs.items():
                x_glob_view[ghosts[off[qq]:off[qq + 1]]] = buf.numpy()

        rng = np.random.default_rng(7)
        x0 = rng.standard_normal(A.n_rows)
        # distributed SpMV against the serial one (same row sums, bitwise)
        xl = np.zeros(A.n_rows)
        xl[mine] = x0[mine]
        refresh(xl)
        y_serial = np.array([np.sum(A.values[A.row_ptr[i]:A.row_ptr[i + 1]] *
                                    x0[A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]]) for i in mine])
        y_dist = np.array([np.sum(A.values[A.row_ptr[i]:A.row_ptr[i + 1]] *
                                  xl[A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]]) for i in mine])
        assert np.array_equal(y_serial, y_dist)
        # all-reduced inner product
        part = torch.tensor([float(np.dot(x0[mine], x0[mine]))], dtype=torch.float64)
        dist.all_reduce(part)
        assert abs(part.item() - float(np.dot(x0, x0))) <= 1e-12 * float(np.dot(x0, x0))
        # block-GS sweep: 4 colour passes with a ghost refresh before each
        t1, t2 = pt.cells_of_points(s.coords, P.depth)
        cell = t2 * P.w + t1
        colour = (t1 & 1) | ((t2 & 1) << 1)
        b = s.b
        colour_rows_all, colour_rows_mine = [], []
        for c in range(4):
            cells_all, cells_mine = [], []
            for cid in np.unique(cell[colour == c]):
                rows = np.nonzero(cell == cid)[0]
                cells_all.append(rows)
                if P.owner[rows[0]] == rank:
                    cells_mine.append(rows)
            colour_rows_all.append(cells_all)
            colour_rows_mine.append(cells_mine)
        x_ser = _colour_pass_serial(Ad, x0, b, P, colour_rows_all)
        xd = np.zeros(A.n_rows)
        xd[mine] = x0[mine]
        for c in range(4):
            refresh(xd)
            r = {tuple(rows): b[rows] - Ad[rows] @ xd for rows in colour_rows_mine[c]}
            for rows in colour_rows_mine[c]:
                xd[rows] = xd[rows] + np.linalg.solve(Ad[np.ix_(rows, rows)], r[tuple(rows)])
        assert np.array_equal(xd[mine], x_ser[mine])
        q.put((rank, "ok"))
    except Exception as e:   # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_exchange_schedule():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
