"""Multi-process (gloo, CPU) test of the z-slab decomposition of the FCN (configs[4]).

Each rank takes its slab geometry from libtn's host planner (tn_fcn_slab_plan),
computes every layer of its slab with the CPU oracle on a halo-extended buffer,
and exchanges the one-plane halos with its neighbours through torch.distributed
send/recv -- the same overlapped, trimmed schedule tn_fcn_forward_slab runs with NCCL on B200: each
layer's interior planes are computed while the previous layer's halo exchange is in flight
(halo planes hold a non-ternary GARBAGE code until received, so an interior plane that read
one would break bit-identity), then the boundary planes, then this layer's exchange of only
the halo sides its consumers read.  The
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


GARBAGE = 5          # a non-ternary code: any read of a halo plane before it arrives shows up


def _post_exchange(buf, rank, world, sides):
    """Start filling buf[0] from rank-1's last owned plane (sides bit 0) and buf[-1] from rank+1's
    first (bit 1), with non-blocking send/recv -- the trimmed exchange tn_fcn_forward_slab posts
    on its comm stream.  Returns the completion (wait + store the received planes)."""
    reqs, got = [], {}
    if rank > 0:
        if sides & 2:
            reqs.append(dist.isend(buf[1].contiguous(), rank - 1))
        if sides & 1:
            got[0] = torch.empty_like(buf[0])
            reqs.append(dist.irecv(got[0], rank - 1))
    if rank + 1 < world:
        if sides & 1:
            reqs.append(dist.isend(buf[-2].contiguous(), rank + 1))
        if sides & 2:
            got[-1] = torch.empty_like(buf[-1])
            reqs.append(dist.irecv(got[-1], rank + 1))

    def finish():
        for r in reqs:
            r.wait()
        for k, v in got.items():
            buf[k] = v
    return finish


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

    # extended codes of the ternarised input, planes [z0-1, z1+1): own planes, halo planes GARBAGE
    # until received (at the volume's ends they stay 0 = the zero padding)
    t, _ = oracle.tern_f32(x, p["t_lo"], p["t_hi"])
    ext = torch.zeros((z1 - z0 + 2,) + x.shape[1:], dtype=torch.int8)
    ext[1:-1] = torch.from_numpy(t[z0:z1])
    if rank > 0:
        ext[0] = GARBAGE
    if rank + 1 < world:
        ext[-1] = GARBAGE
    x_sides = 3 if table[0][2] == 1 else 1
    fin_x = _post_exchange(ext, rank, world, x_sides)
    bufs = {-1: ext[None]}                                        # tensor -> [c][planes z-1 .. z1][h][w]
    firsts = {-1: z0 - 1}
    pending = fin_x                                               # the exchange in flight
    acts = {}
    for i, (kind, co, s, segs) in enumerate(table):
        L = plan[i]
        assert L.c == co
        dz = L.z1 - L.z0

        def planes(a, b):
            """Codes of owned output planes [a, b) (local) from the current input buffers."""
            parts = []
            for (src, up) in segs:
                a5 = bufs[src].numpy()[None]                      # NCDHW
                first = firsts[src]
                if up:
                    a5 = oracle.upsample2(a5)
                    first = 2 * first
                lo_plane = (L.z0 + a) * s - 1                     # conv-input planes needed
                n_in = (b - a - 1) * s + 3
                parts.append(a5[:, :, lo_plane - first: lo_plane - first + n_in])
            inp = np.concatenate(parts, axis=1) if len(parts) > 1 else parts[0]
            acc = oracle.conv3d(np.ascontiguousarray(inp), p["weights"][i], stride=s, pad=(0, 1, 1))
            assert acc.shape[2] == b - a, (i, acc.shape, a, b)
            return oracle.requant(acc, p["lo"][i], p["hi"][i])[0]

        # plane-major buffer [planes][c][h][w]; halo planes GARBAGE until received
        pm = torch.zeros((dz + 2, co, L.h, L.w), dtype=torch.int8)
        # the overlapped schedule: interior planes while the previous layer's halos are still in
        # flight (they hold GARBAGE), then the boundary planes once that exchange completed
        if dz > 2:
            pm[2:dz] = torch.from_numpy(planes(1, dz - 1)).permute(1, 0, 2, 3)
        pending()
        pm[1] = torch.from_numpy(planes(0, 1))[:, 0]
        if dz > 1:
            pm[dz] = torch.from_numpy(planes(dz - 1, dz))[:, 0]
        acts[i] = pm[1:-1].permute(1, 0, 2, 3).numpy().copy()
        if L.halo:
            if rank > 0 and (L.halo & 1):
                pm[0] = GARBAGE
            if rank + 1 < world and (L.halo & 2):
                pm[-1] = GARBAGE
            fin = _post_exchange(pm, rank, world, L.halo)

            def pending(pm=pm, fin=fin, i=i):
                fin()
                bufs[i] = pm.permute(1, 0, 2, 3).contiguous()
        else:
            pending = (lambda: None)
        bufs[i] = pm.permute(1, 0, 2, 3).contiguous()
        firsts[i] = L.z0 - 1
    pending()
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
    # halo sides (bit 0 lower, bit 1 upper): every R9 tensor feeds a stride-1 consumer (the skips
    # #2/#4/#6 also feed the stride-2 #3/#5/#7), so both sides; the last one feeds only A8
    assert plan[-1].halo == 0 and all(L.halo == 3 for L in plan[:-1])
    assert plan[0].plane_bytes == 512 * 512 * 8 and plan[5].plane_bytes == 128 * 128 * 16
    # slab bounds must be multiples of the total downsampling (8)
    st = tn.lib.tn_fcn_slab_plan(h, tn.dims(1, 1, 256, 512, 512), 4, 96, None, 0, None)
    assert st == tn.TN_ESHAPE


def test_slab_plan_trims_halo_sides():
    """A tensor whose only consumer is a stride-2 conv exchanges only its lower halo plane (slab
    starts are even, so output z reads input planes 2z-1..2z+1 and never the plane above)."""
    import paper_1801_09449_b200 as tn
    F, C = tn.TN_LAYER_FIRST, tn.TN_LAYER_CONV
    table = [(F, 16, 1, [(-1, 0)]), (C, 16, 2, [(0, 0)]), (C, 16, 1, [(1, 0)]), (C, 16, 1, [(2, 0)])]
    layers = (tn.tn_layer * len(table))()
    for i, (kind, co, s_, segs) in enumerate(table):
        L = layers[i]
        L.kind, L.c_out, L.stride, L.dil, L.nseg = kind, co, s_, 1, len(segs)
        for j, (src, up) in enumerate(segs):
            L.src[j], L.upsample[j], L.wp[j] = src, up, 0x1000
        L.lo = L.hi = 0x1000
    h = ctypes.c_void_p()
    P = ctypes.c_void_p(0x1000)
    assert tn.lib.tn_fcn_create(layers, len(table), -200.0, 200.0, P, P, 2, ctypes.byref(h)) == 0
    plan = _plan(tn, h, len(table), (1, 1, 16, 8, 8), 4, 8)
    assert [L.halo for L in plan] == [1, 3, 3, 0]
    tn.lib.tn_fcn_destroy(h)
