"""Multi-process (gloo, CPU) test of the z-slab decomposition of the FCN (configs[4]).

Each rank takes its slab geometry from libtn's host planner (tn_fcn_slab_plan),
computes every layer of its slab with the CPU oracle on a halo-extended buffer,
and exchanges the one-plane halos with its neighbours through torch.distributed
send/recv -- the same schedule tn_fcn_forward_slab runs with NCCL on B200.  The
gathered logits must equal the whole-volume oracle bit for bit.  (The CUDA slab
kernels and offsets are covered on the GPU by tn_fcn_forward_slabs_local.)
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dummy_net(tn):
    """A tn_fcn handle with placeholder device pointers: the planner only reads shapes."""
    table = tn.fcn_table()
    layers = (tn.tn_layer * len(table))()
    for i, (kind, co, s, segs) in enumerate(table):
        L = layers[i]
        L.kind, L.c_out, L.stride, L.dil, L.nseg = kind, co, s, 1, len(segs)
        for j, (src, up) in enumerate(segs):
            L.src[j], L.upsample[j], L.wp[j] = src, up, 0x1000
        L.lo = L.hi = 0x1000
    h = ctypes.c_void_p()
    P = ctypes.c_void_p(0x1000)
    assert tn.lib.tn_fcn_create(layers, len(table), -200.0, 200.0, P, P, 2, ctypes.byref(h)) == 0
    return h, table


def _plan(tn, h, n_layers, shape, z0, z1):
    arr = (tn.tn_slab_layer * n_layers)()
    nb = ctypes.c_size_t()
    st = tn.lib.tn_fcn_slab_plan(h, tn.dims(*shape), z0, z1, arr, n_layers, ctypes.byref(nb))
    assert st == 0, tn.lib.tn_last_error()
    return list(arr)


def _exchange(buf, rank, world):
    """Fill buf[0] from rank-1's last owned plane and buf[-1] from rank+1's first."""
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(buf[1].contiguous(), rank - 1))
        lo = torch.empty_like(buf[0])
        reqs.append(dist.irecv(lo, rank - 1))
    if rank + 1 < world:
        reqs.append(dist.isend(buf[-2].contiguous(), rank + 1))
        hi = torch.empty_like(buf[-1])
        reqs.append(dist.irecv(hi, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        buf[0] = lo
    if rank + 1 < world:
        buf[-1] = hi


def _worker(rank, world, port, shape, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    import paper_1801_09449_b200 as tn

    h, table = _dummy_net(tn)
    D = shape[2]
    z0, z1 = rank * D // world, (rank + 1) * D // world
    plan = _plan(tn, h, len(table), shape, z0, z1)
    p = synth.fcn_params()
    x = synth.ct_volume(shape, seed=3)[0, 0]                      # [D][H][W]

    # extended codes of the ternarised input, planes [z0-1, z1+1); outside -> 0
    t, _ = oracle.tern_f32(x, p["t_lo"], p["t_hi"])
    ext = torch.zeros((z1 - z0 + 2,) + x.shape[1:], dtype=torch.int8)
    ext[1:-1] = torch.from_numpy(t[z0:z1])
    _exchange(ext, rank, world)
    bufs = {-1: (ext, z0 - 1)}                                    # layer -> (buffer [c?][planes], first plane)
    acts = {}
    for i, (kind, co, s, segs) in enumerate(table):
        L = plan[i]
        assert L.c == co
        parts = []
        for (src, up) in segs:
            b, b0 = bufs[src]
            a = b.numpy()
            if a.ndim == 3:
                a = a[None]                                       # [1][planes][h][w]
            a = a[None]                                           # NCDHW
            if up:
                a = oracle.upsample2(a)
                first = 2 * b0
            else:
                first = b0
            lo_plane = L.z0 * s - 1                               # conv-input planes needed
            n_in = (L.z1 - L.z0 - 1) * s + 3
            parts.append(a[:, :, lo_plane - first: lo_plane - first + n_in])
        inp = np.concatenate(parts, axis=1) if len(parts) > 1 else parts[0]
        acc = oracle.conv3d(np.ascontiguousarray(inp), p["weights"][i], stride=s, pad=(0, 1, 1))
        assert acc.shape[2] == L.z1 - L.z0, (i, acc.shape, L.z0, L.z1)
        codes = oracle.requant(acc, p["lo"][i], p["hi"][i])[0]   # [co][planes][h][w]
        out = torch.zeros((co, L.z1 - L.z0 + 2) + codes.shape[2:], dtype=torch.int8)
        out[:, 1:-1] = torch.from_numpy(codes)
        if L.halo:
            # exchange plane-major views: move the plane axis first
            pm = out.permute(1, 0, 2, 3).contiguous()
            _exchange(pm, rank, world)
            out = pm.permute(1, 0, 2, 3).contiguous()
            # global-boundary halos stay zero (= the convolution's zero padding)
        bufs[i] = (out, L.z0 - 1)
        acts[i] = codes
    logits = oracle.predict(np.ascontiguousarray(acts[len(table) - 1][None]), p["pred_w"], p["pred_b"])
    gathered = [torch.empty(0)] * world
    dist.all_gather_object(gathered, (z0, z1, logits))
    if rank == 0:
        out_q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (1, 1, 16, 16, 24)), (4, (1, 1, 32, 16, 16))])
def test_slab_decomposition_matches_whole_volume(world, shape):
    import oracle
    import synth
    p = synth.fcn_params()
    x = synth.ct_volume(shape, seed=3)
    ref, _, _ = oracle.fcn_forward(x, p["t_lo"], p["t_hi"], p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    gathered = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    got = np.zeros_like(ref)
    for (z0, z1, lg) in gathered:
        got[:, :, z0:z1] = lg
    np.testing.assert_array_equal(got, ref)


def test_slab_plan_geometry():
    import paper_1801_09449_b200 as tn
    h, table = _dummy_net(tn)
    plan = _plan(tn, h, len(table), (1, 1, 256, 512, 512), 64, 96)
    scales = [L.level_scale for L in plan]
    assert scales == [1, 1, 2, 2, 4, 4, 8, 8, 4, 4, 2, 2, 1, 1]
    assert [(L.z0, L.z1) for L in plan][:7] == [(64, 96), (64, 96), (32, 48), (32, 48), (16, 24), (16, 24), (8, 12)]
    assert plan[-1].halo == 0 and all(L.halo == 1 for L in plan[:-1])
    assert plan[0].plane_bytes == 512 * 512 * 8 and plan[5].plane_bytes == 128 * 128 * 16
    # slab bounds must be multiples of the total downsampling (8)
    st = tn.lib.tn_fcn_slab_plan(h, tn.dims(1, 1, 256, 512, 512), 4, 96, None, 0, None)
    assert st == tn.TN_ESHAPE
