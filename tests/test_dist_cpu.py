"""CPU (gloo, world_size 2 and 3) check of the slab decomposition's host-side protocol
(include/airebo_b200.h, ab_create_dist).

Each process plays one rank: ownership and slab bounds come from the real library's host-only
calls (ab_slab_of, ab_slab_info); the halo rule, the channel / image-shift convention and the
exchange order of the engine (send left, recv right, send right, recv left; with two ranks both
messages go to the same peer and match in issue order) are replayed with torch.distributed send /
recv over gloo.  Checked against brute force on the global periodic system:
  * every atom is owned by exactly one rank, inside its slab;
  * the ghost instances a rank holds (x halo from the neighbours + y/z images) are exactly the
    atom images inside its padded slab region -- nothing missing, nothing duplicated;
  * reverse communication returns every ghost contribution to the owner exactly once;
  * the ownership rule (lower instance key computes the term) counts every LJ half pair within
    r_c once over all ranks (total = the oracle's half list);
  * bench.py's max-over-ranks reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RC_MAX, SKIN = 10.2, 1.0  # toy_ch.param: LJ cutoff 3 sigma_CC, skin (halo h = r_c,max + skin)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _key(g, s):
    return (int(g), int(s[0]), int(s[1]), int(s[2]))


def _exchange(rank, ws, send0, send1):
    """Engine order: send(left) recv(right) send(right) recv(left); counts first, then payload."""
    left, right = (rank - 1) % ws, (rank + 1) % ws
    c = [torch.tensor([len(send0)], dtype=torch.int64), torch.tensor([len(send1)], dtype=torch.int64)]
    r = [torch.zeros(1, dtype=torch.int64), torch.zeros(1, dtype=torch.int64)]
    reqs = [dist.isend(c[0], left), dist.irecv(r[1], right), dist.isend(c[1], right), dist.irecv(r[0], left)]
    for q in reqs:
        q.wait()
    p_s = [torch.from_numpy(np.ascontiguousarray(send0, dtype=np.float64)).reshape(-1),
           torch.from_numpy(np.ascontiguousarray(send1, dtype=np.float64)).reshape(-1)]
    w = send0.shape[1] if len(send0) else send1.shape[1] if len(send1) else 1
    p_r = [torch.zeros(int(r[0]) * w, dtype=torch.float64), torch.zeros(int(r[1]) * w, dtype=torch.float64)]
    reqs = []
    if p_s[0].numel():
        reqs.append(dist.isend(p_s[0], left))
    if p_r[1].numel():
        reqs.append(dist.irecv(p_r[1], right))
    if p_s[1].numel():
        reqs.append(dist.isend(p_s[1], right))
    if p_r[0].numel():
        reqs.append(dist.irecv(p_r[0], left))
    for q in reqs:
        q.wait()
    return p_r[0].numpy().reshape(-1, w), p_r[1].numpy().reshape(-1, w)


def _worker(rank, ws, port, reps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_1810_07026_b200 import engine as E
        from paper_1810_07026_b200 import inputs as I
        import bench
        s = I.polyethylene(reps, 0.03, 7, 8)
        L = s.box
        h = RC_MAX + SKIN
        n = s.n
        x = I.wrap(s.x, L)
        xlo, xhi, ok = E.slab_info(L, h, ws, rank)
        assert ok
        owner = np.array([E.slab_of(v, L[0], ws) for v in x[:, 0]])
        loc = np.nonzero(owner == rank)[0]
        assert np.all((x[loc, 0] >= xlo) & (x[loc, 0] < xhi))
        # ---- halo: channel 0 = left face -> left neighbour, channel 1 = right face -> right
        s0 = loc[x[loc, 0] < xlo + h]
        s1 = loc[x[loc, 0] >= xhi - h]
        rec = lambda idx: np.column_stack([idx.astype(np.float64), x[idx]])
        r0, r1 = _exchange(rank, ws, rec(s0), rec(s1))
        sx = [-1 if rank == 0 else 0, 1 if rank == ws - 1 else 0]
        inst = {}  # instance key -> (position, base key); bases: locals + x ghosts
        xchan = {}  # x-ghost key -> channel it arrived on
        bases = []
        for i in loc:
            bases.append((_key(i, (0, 0, 0)), x[i]))
        for c, rr in enumerate((r0, r1)):
            for row in rr:
                g = int(row[0])
                p = row[1:].copy()
                p[0] = p[0] + sx[c] * L[0]
                k = _key(g, (sx[c], 0, 0))
                assert k not in inst, "duplicate x ghost"
                inst[k] = (p, k)
                xchan[k] = c
                bases.append((k, p))
        smax = [int(np.ceil(h / L[d])) for d in range(3)]
        lo = np.array([xlo - h, -h, -h])
        hi = np.array([xhi + h, L[1] + h, L[2] + h])
        for kb, p in bases:
            for sy in range(-smax[1], smax[1] + 1):
                for sz in range(-smax[2], smax[2] + 1):
                    if sy == 0 and sz == 0:
                        continue
                    u = p + np.array([0.0, sy * L[1], sz * L[2]])
                    if np.all(u >= lo) and np.all(u < hi):
                        k = (kb[0], kb[1], sy, sz)
                        assert k not in inst, "duplicate image"
                        inst[k] = (u, kb)
        # ---- brute force: every image of every atom inside the padded region, locals excluded
        want = set()
        for g in range(n):
            for a in range(-1, 2):
                for b in range(-smax[1], smax[1] + 1):
                    for c in range(-smax[2], smax[2] + 1):
                        if owner[g] == rank and a == 0 and b == 0 and c == 0:
                            continue
                        u = x[g] + np.array([a * L[0], b * L[1], c * L[2]])
                        if np.all(u >= lo) and np.all(u < hi):
                            want.add((g, a, b, c))
        assert set(inst) == want, (len(inst), len(want), sorted(set(inst) ^ want)[:5])
        # ---- reverse communication of ghost "forces" f(g, s): an image adds into its base (a
        # local atom: folded here; an x ghost: accumulated and sent back on its channel)
        f = lambda k: np.array([1.0 + k[0], 0.01 * (k[1] + 2) + 0.001 * (k[2] + 3) + 1e-4 * (k[3] + 5), 1.0])
        local_keys = {_key(i, (0, 0, 0)) for i in loc}
        Fl = {int(i): np.zeros(3) for i in loc}
        Fx = {k: np.zeros(3) for k in xchan}
        for k, (_, kb) in inst.items():
            if kb in local_keys:
                Fl[kb[0]] += f(k)
            else:
                Fx[kb] += f(k)
        back = [np.array([np.concatenate([[k[0]], Fx[k]]) for k in xchan if xchan[k] == c]).reshape(-1, 4)
                for c in (0, 1)]
        b0, b1 = _exchange(rank, ws, back[0], back[1])
        for row in np.concatenate([b0, b1]):
            Fl[int(row[0])] += row[1:]
        tot = np.zeros((n, 3))
        for i, v in Fl.items():
            tot[i] = v
        tt = torch.from_numpy(tot)
        dist.all_reduce(tt)
        # every instance of every atom in every rank's halo, once
        exp = np.zeros((n, 3))
        allk = [None] * ws
        dist.all_gather_object(allk, sorted(inst))
        for ks in allk:
            for k in ks:
                exp[k[0]] += f(k)
        assert np.allclose(tt.numpy(), exp, rtol=0, atol=1e-9)
        # ---- ownership rule: LJ half pairs within r_c counted once globally
        pos = {_key(i, (0, 0, 0)): x[i] for i in loc}
        pos.update({k: v[0] for k, v in inst.items()})
        rc = {0: 10.2, 1: 9.0, 2: 7.8}  # lj.CC.rc, lj.CH.rc, lj.HH.rc of params/toy_ch.param
        keys = np.array(list(pos.keys()))
        P = np.array([pos[tuple(k)] for k in keys])
        cnt = 0
        for i in loc:
            d = P - x[i]
            r2 = (d * d).sum(1)
            for q in np.nonzero(r2 <= 10.2 ** 2)[0]:
                k = tuple(keys[q])
                if k == _key(i, (0, 0, 0)):
                    continue
                if k > _key(i, (0, 0, 0)) and r2[q] <= rc[s.types[i] + s.types[k[0]]] ** 2:
                    cnt += 1
        ct = torch.tensor([cnt], dtype=torch.int64)
        dist.all_reduce(ct)
        # bench.py's timing reduction: max over ranks
        mx = bench.reduce_max(float(rank + 1), ws)
        out[rank] = (int(ct.item()), mx, len(loc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws,reps", [(2, (4, 2, 4)), (3, (5, 2, 4))])
def test_slab_protocol_gloo(ws, reps):
    from oracle import oracle as O
    from paper_1810_07026_b200 import build
    from paper_1810_07026_b200 import inputs as I
    build.build()
    port = _free_port()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(ws, port, reps, out), nprocs=ws, start_method="spawn", join=True)
    s = I.polyethylene(reps, 0.03, 7, 8)
    n_half = len(O.get_list(s.types, s.x, s.box, 2))
    assert sum(out[r][2] for r in range(ws)) == s.n
    for r in range(ws):
        assert out[r][0] == n_half, (out[r][0], n_half)
        assert out[r][1] == float(ws)
