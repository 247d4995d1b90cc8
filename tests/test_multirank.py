"""Multi-rank host logic on CPU (gloo): the horizontal block decomposition planned by the
product (tpmg_plan_decomposition) plus the face-halo protocol of tpmg_host.cpp:exchange()
(pack [W|E|S|N] like k_pack_faces; send W->west, E->east, recv E<-east, W<-west, then S/N,
matched in order per peer exactly like an NCCL group) must reproduce the global operator
apply bit for bit on every tile, and the all-reduced dot product must match the global one.
Runs world_size 2 (2x1: W and E neighbours coincide) and 4 (2x2)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tile_apply(u, halo, co, nz):
    """numpy restatement of the apply kernel on one tile with face halos (same op order)."""
    nzz, ny, nx = u.shape
    bv, sv, av = co["bv"], co["sv"], co["av"]
    uw = np.concatenate([halo["W"][:, :, None], u[:, :, :-1]], axis=2)
    ue = np.concatenate([u[:, :, 1:], halo["E"][:, :, None]], axis=2)
    us = np.concatenate([halo["S"][:, None, :], u[:, :-1, :]], axis=1)
    un = np.concatenate([u[:, 1:, :], halo["N"][:, None, :]], axis=1)
    y = np.empty_like(u)
    for k in range(nz):
        upper = -(av[k + 1] * co["ah"])
        lower = -(av[k] * co["ah"])
        nw, ne, ns, nn = (-(sv[k] * co[d]) for d in ("sw", "se", "ss", "sn"))
        diag = bv[k] * co["bh"] - ((upper + lower) + (((nw + ne) + ns) + nn))
        v = diag * u[k]
        if k + 1 < nz:
            v = v + upper * u[k + 1]
        if k > 0:
            v = v + lower * u[k - 1]
        v = v + nw * uw[k]
        v = v + ne * ue[k]
        v = v + ns * us[k]
        v = v + nn * un[k]
        y[k] = v
    return y


def _worker(rank, world, px, py, port, q):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import ctypes as C

    import torch

    import oracle as O
    from paper_1408_2981_b200 import _capi, synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        NX, NY, NZ = 32, 16, 6
        P = synth.make_problem(NX, NY, NZ, omega2=1e-2, lambda2=1e-2, grading="quadratic",
                               profile="uniform", profile_seed=7, depth=3)
        L = _capi.load("exact")
        n = C.c_int()
        arrs = [(C.c_int64 * 8)() for _ in range(4)]
        nbr = (C.c_int * 4)()
        assert L.tpmg_plan_decomposition(NX, NY, px, py, rank, P.depth, 8, C.byref(n), *arrs, nbr) == 0
        lvl = n.value - 1
        tnx, tny, x0, y0 = (int(a[lvl]) for a in arrs)
        # global oracle + its hatted coefficients, extracted to the tile like tpmg_hier_create
        o = O.OracleHierarchy.from_problem(P)
        co = o.coefficients(o.finest)
        se = co["sh"][: NX * NY].reshape(NY, NX)
        sn = co["sh"][NX * NY:].reshape(NY, NX)
        js, is_ = np.arange(y0, y0 + tny), np.arange(x0, x0 + tnx)
        tile = {"bh": co["bh"].reshape(NY, NX)[np.ix_(js, is_)],
                "ah": co["ah"].reshape(NY, NX)[np.ix_(js, is_)],
                "se": se[np.ix_(js, is_)], "sn": sn[np.ix_(js, is_)],
                "sw": se[np.ix_(js, (is_ - 1) % NX)], "ss": sn[np.ix_((js - 1) % NY, is_)],
                "bv": co["bv"], "sv": co["sv"], "av": co["av"]}
        u_glob = np.random.default_rng(3).standard_normal((NZ, NY, NX))
        u = np.ascontiguousarray(u_glob[:, y0:y0 + tny, x0:x0 + tnx])
        # pack faces exactly like k_pack_faces: W,E as [k][j], S,N as [k][i]
        faces = {"W": u[:, :, 0], "E": u[:, :, -1], "S": u[:, 0, :], "N": u[:, -1, :]}
        halo = {}
        west, east, south, north = list(nbr)
        ops = []
        recv = {d: torch.empty(faces[o_].shape, dtype=torch.float64) for d, o_ in
                (("E", "W"), ("W", "E"), ("N", "S"), ("S", "N"))}
        if px > 1:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(faces["W"])), west),
                    dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(faces["E"])), east),
                    dist.P2POp(dist.irecv, recv["E"], east),
                    dist.P2POp(dist.irecv, recv["W"], west)]
        if py > 1:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(faces["S"])), south),
                    dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(faces["N"])), north),
                    dist.P2POp(dist.irecv, recv["N"], north),
                    dist.P2POp(dist.irecv, recv["S"], south)]
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        # dimensions with one rank wrap onto the tile itself (self_halo)
        halo["W"] = recv["W"].numpy() if px > 1 else u[:, :, -1]
        halo["E"] = recv["E"].numpy() if px > 1 else u[:, :, 0]
        halo["S"] = recv["S"].numpy() if py > 1 else u[:, -1, :]
        halo["N"] = recv["N"].numpy() if py > 1 else u[:, 0, :]
        y_tile = _tile_apply(u, halo, tile, NZ)
        y_glob = o.apply(o.finest, synth.x_fastest_to_k_fastest(u_glob))
        y_ref = synth.k_fastest_to_x_fastest(y_glob, NX, NY, NZ)[:, y0:y0 + tny, x0:x0 + tnx]
        bitwise = bool(np.array_equal(y_tile, y_ref))
        # global dot through the all-reduce
        part = torch.tensor([float(np.dot(u.reshape(-1), y_tile.reshape(-1)))], dtype=torch.float64)
        dist.all_reduce(part)
        dref = float(np.dot(u_glob.reshape(-1), synth.k_fastest_to_x_fastest(y_glob, NX, NY, NZ).reshape(-1)))
        q.put((rank, bitwise, abs(part.item() - dref) / abs(dref), (tnx, tny, x0, y0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("px,py", [(2, 1), (2, 2), (1, 2)])
def test_tiles_and_halo_protocol_reproduce_global_apply(px, py):
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, px, py, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tiles = set()
    for rank, bitwise, dot_err, t in res:
        assert bitwise, f"rank {rank}: tile apply differs from the global operator"
        assert dot_err <= 1e-13
        tiles.add(t)
    assert len(tiles) == world  # disjoint tiles


# ---- the two-cell halo with corners (tpmg_host.cpp:exchange_deep, tpmg::Halo2) ----------------
DDX = (-1, 1, 0, 0, -1, 1, -1, 1)   # pieces W, E, S, N, SW, SE, NW, NE (kDeepDx / kDeepDy)
DDY = (0, 0, -1, 1, -1, -1, 1, 1)
OPP = (1, 0, 3, 2, 7, 6, 5, 4)       # kOpp: piece d lands in the receiver's slot OPP[d]


def _deep_pieces(u):
    """k_pack_deep's pieces: W/E [k][j][c] from columns c / nx-2+c, S/N [k][r][i] from rows
    r / ny-2+r, corners [k][r][c] from the 2x2 corner blocks."""
    return [np.ascontiguousarray(a) for a in (
        u[:, :, 0:2], u[:, :, -2:], u[:, 0:2, :], u[:, -2:, :],
        u[:, 0:2, 0:2], u[:, 0:2, -2:], u[:, -2:, 0:2], u[:, -2:, -2:])]


def _halo2_window(u, slots, xs, ys):
    """The (nz, ny+4, nx+4) block halo2_at reads: inside from u, outside from the slots
    (W2, E2, S2, N2, SW, SE, NW, NE), a dimension with one rank wrapping onto the tile."""
    nz, ny, nx = u.shape
    out = np.empty((nz, ny + 4, nx + 4))
    for gy in range(-2, ny + 2):
        for gx in range(-2, nx + 2):
            x, y = gx, gy
            if not xs:
                x %= nx
            if not ys:
                y %= ny
            ox = -1 if x < 0 else (1 if x >= nx else 0)
            oy = -1 if y < 0 else (1 if y >= ny else 0)
            c = x + 2 if ox < 0 else x - nx
            r = y + 2 if oy < 0 else y - ny
            if ox == 0 and oy == 0:
                v = u[:, y, x]
            elif oy == 0:
                v = slots[0 if ox < 0 else 1][:, y, c]
            elif ox == 0:
                v = slots[2 if oy < 0 else 3][:, r, x]
            else:
                v = slots[4 + (0 if oy < 0 else 2) + (0 if ox < 0 else 1)][:, r, c]
            out[:, gy + 2, gx + 2] = v
    return out


def _deep_worker(rank, world, px, py, port, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        NX, NY, NZ = 16 * px, 8 * py, 3
        tnx, tny = NX // px, NY // py
        rx, ry = rank % px, rank // px
        x0, y0 = rx * tnx, ry * tny
        u_glob = np.random.default_rng(11).standard_normal((NZ, NY, NX))
        u = np.ascontiguousarray(u_glob[:, y0:y0 + tny, x0:x0 + tnx])
        xs, ys = px > 1, py > 1
        live = [(DDX[d] == 0 or xs) and (DDY[d] == 0 or ys) for d in range(8)]
        nbr = [((ry + DDY[d]) % py) * px + (rx + DDX[d]) % px for d in range(8)]
        pieces = _deep_pieces(u)
        slots = [np.zeros_like(p) for p in (pieces[1], pieces[0], pieces[3], pieces[2],
                                            pieces[7], pieces[6], pieces[5], pieces[4])]
        recv = [torch.from_numpy(s) for s in slots]
        ops = []
        for d in range(8):  # exchange_deep's NCCL group: send d, receive slot OPP[d]
            if not live[d]:
                continue
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(pieces[d]), nbr[d]))
            ops.append(dist.P2POp(dist.irecv, recv[OPP[d]], nbr[OPP[d]]))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        win = _halo2_window(u, [r.numpy() for r in recv], xs, ys)
        ref = np.take(np.take(u_glob, np.arange(y0 - 2, y0 + tny + 2) % NY, axis=1),
                      np.arange(x0 - 2, x0 + tnx + 2) % NX, axis=2)
        q.put((rank, bool(np.array_equal(win, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2), (4, 2)])
def test_deep_halo_protocol_reproduces_the_periodic_window(px, py):
    """The decomposed fused residual + restriction's exchange (8 pieces, sends in the order
    W,E,S,N,SW,SE,NW,NE, receives into the opposite slots in the same order, so that pieces two
    ranks exchange in several directions -- px or py = 2, where W = E and all diagonals coincide
    -- match like an NCCL group) gives every tile the global field two cells beyond it."""
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_deep_worker, args=(r, world, px, py, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
