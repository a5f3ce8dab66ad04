"""CPU, world_size 2 over gloo: the landmark-sharded multi-GPU decomposition.

Each rank owns the landmark shard that ``shard.plan_shards`` assigns it and
computes its partial camera-space quantities (the per-term S'.v partial, the
U / b_p partial sums, the cost partial) -- here with the CPU oracle standing in
for the device kernels, since this container has no GPU.  The partials are
summed with an allreduce exactly where libpovar.so calls ncclAllReduce, and
must reproduce the unsharded result; the power-series stop decisions taken on
the reduced vectors must agree on both ranks.  The NCCL unique-id broadcast
used by bench.py / DeviceProblem is exercised too.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sub_graph(O, pr, lo, hi):
    keep = (pr.landmark_indices >= lo) & (pr.landmark_indices < hi)
    return O.make_graph(pr.num_cameras, pr.num_landmarks, pr.camera_indices[keep],
                        pr.landmark_indices[keep], pr.measurements[keep])


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import _kat
        from oracle import povar_oracle as O
        from paper_2405_05079_b200 import shard

        pr, st = _kat.long_track_case()
        plan = shard.plan_shards(pr, world)
        lo, hi = plan[rank]
        g_loc = _sub_graph(O, pr, lo, hi)
        g_all = O.graph_of(pr)
        lam = 1e-3

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        # per LM iteration: U_raw and b_p partials -> allreduce (povar.cu op_linearize)
        lin = O.linearize(g_loc, st.cameras, st.landmarks, 1)
        loc = O.assemble(g_loc, lin, lam, False)
        U_sum = allreduce(loc.U_raw)
        bp_sum = allreduce(loc.b_p)
        ref = O.assemble(g_all, O.linearize(g_all, st.cameras, st.landmarks, 1), lam, False)
        ok = [np.allclose(U_sum, ref.U_raw, rtol=1e-12, atol=1e-12),
              np.allclose(bp_sum, ref.b_p, rtol=1e-12, atol=1e-12)]
        # per term: partial W V+ W^T v -> allreduce (povar.cu launch_cam_term)
        v = np.random.default_rng(7).standard_normal(pr.num_cameras * 12)
        y = allreduce(O.coupling(loc, v))
        ok.append(np.allclose(y, O.coupling(ref, v), rtol=1e-11, atol=1e-11))
        # replicated stop test on the reduced vectors: identical decision on every rank
        U_inv = np.linalg.inv(O.jacobi_damp(U_sum, lam))
        t = np.einsum("nij,nj->ni", U_inv, y.reshape(-1, 12))
        ratio = np.linalg.norm(t) / max(np.linalg.norm(v), 1e-300)
        dec = torch.tensor([ratio], dtype=torch.float64)
        mx, mn = dec.clone(), dec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        ok.append(float(mx) == float(mn))
        # cost partials -> allreduce (povar.cu op_cost)
        f = allreduce(np.array([O.total_cost(g_loc, st.cameras, st.landmarks, 1)]))[0]
        ok.append(abs(f - O.total_cost(g_all, st.cameras, st.landmarks, 1)) <= 1e-12 * f)
        # PCG (povar.cu op_pcg): the block-diagonal moments and every S'.p partial are
        # allreduced; the CG recurrences run replicated on the reduced camera vectors
        full = ref
        U_d = O.jacobi_damp(U_sum, lam)
        contrib = allreduce(loc.U - O.schur_diag_blocks(loc))
        m_inv = np.linalg.inv(U_d - contrib)
        b_l_part = loc.b_l  # landmark-local
        rhs = -(bp_sum.ravel() - allreduce(O.w_apply(loc, np.einsum("nij,nj->ni", loc.V_pinv,
                                                                      b_l_part)).ravel()))
        n = pr.num_cameras

        def mapply(M, v):
            return np.einsum("nij,nj->ni", M, v.reshape(n, -1)).ravel()

        x = np.zeros_like(rhs)
        r = rhs.copy()
        z = mapply(m_inv, r)
        p = z.copy()
        rz = float(r @ z)
        its = 0
        rhs_norm = np.linalg.norm(rhs)
        for it in range(1, 200):
            its = it
            sp = mapply(U_d, p) - allreduce(O.coupling(loc, p))
            alpha = rz / float(p @ sp)
            x += alpha * p
            r -= alpha * sp
            if np.linalg.norm(r) / rhs_norm <= 1e-8:
                break
            z = mapply(m_inv, r)
            rz_new = float(r @ z)
            p = z + (rz_new / rz) * p
            rz = rz_new
        want = O.pcg_solve(full, 199, 1e-8)
        ok.append(abs(its - want.iterations) <= 1)
        ok.append(np.linalg.norm(x - want.pose_update) <= 1e-6 * np.linalg.norm(want.pose_update))
        got = torch.tensor([float(its)], dtype=torch.float64)
        mx, mn = got.clone(), got.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        ok.append(float(mx) == float(mn))  # identical stop decision on every rank
        # NCCL id broadcast used to build the device communicator
        nid = shard.broadcast_nccl_id(rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        ok.append(len(nid) == 128 and all(i == ids[0] for i in ids))
        q.put((rank, ok, plan))
    except Exception as exc:  # report instead of leaving the parent waiting on the queue
        q.put((rank, [repr(exc)], None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shard_partials_allreduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, plan in results:
        assert all(isinstance(x, (bool, np.bool_)) and x for x in ok), (rank, ok)
    assert results[0][2] == results[1][2]
