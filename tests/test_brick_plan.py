"""Host logic of the brick kernels (csrc/persist_brick.cuh: brick_geometry, through phipm_brick_plan): every
decomposition it returns must tile the grid so that each row belongs to exactly one (CTA, warp, lane, plane),
fit the hardware limits the kernels assume, and stage exactly the planes the marching warps wait for."""
import numpy as np
import pytest

import paper_0907_4631_b200 as P

SMEM = 219 * 1024
GRIDS = [(128, 128, 128), (64, 256, 128), (192, 96, 96), (96, 96, 96), (20, 22, 30), (72, 70, 68), (250, 9, 11),
         (64, 37, 29), (2, 5, 7), (128, 20, 24), (252, 100, 80), (64, 64, 128), (6, 1, 1), (128, 128, 40)]


@pytest.mark.parametrize("nx,ny,nz", GRIDS)
def test_plan_limits_and_exact_cover(nx, ny, nz):
    g = P.brick_plan(nx, ny, nz, 148, SMEM)
    assert g is not None
    assert g["py"] * g["pz"] <= 148                              # one CTA per SM
    assert g["nseg"] == -(-nx // 64) and g["ncol"] == g["nseg"] * g["ylen"] <= 32
    assert g["ngrp"] == 32 // g["ncol"] >= 1 and 1 <= g["ppg"] <= 8      # 8 TMEM pair slots per thread
    assert g["zlen"] <= g["ngrp"] * g["ppg"]
    assert g["lstride"] == nx + 4 and g["pstride"] % 16 == 0 and g["pstride"] >= (g["ylen"] + 2) * g["lstride"]
    assert (g["zlen"] + 2) * g["pstride"] * 8 <= SMEM and g["zlen"] + 2 <= 36
    assert nx + 4 <= 256 and g["ylen"] + 2 <= 256                # tensor-map box limits
    # the kernels' index mapping, replayed: CTA -> brick, warp -> (segment, line, z group), lane -> x pair
    owner = np.zeros((nz, ny, nx), dtype=np.int32)
    for cta in range(g["py"] * g["pz"]):
        by, bz = cta % g["py"], cta // g["py"]
        y0, z0 = by * g["ylen"], bz * g["zlen"]
        zl = min(g["zlen"], nz - z0)
        assert zl >= 1 and y0 < ny                               # no empty brick
        for warp in range(32):
            col, grp = warp % g["ncol"], warp // g["ncol"]
            seg, yl = col % g["nseg"], col // g["nseg"]
            yy, zb = y0 + yl, grp * g["ppg"]
            cnt = max(0, min(g["ppg"], zl - zb)) if (grp < g["ngrp"] and yy < ny) else 0
            x0, x1 = seg * 64, min(nx, seg * 64 + 64)
            if cnt and x0 < x1:
                owner[z0 + zb:z0 + zb + cnt, yy, x0:x1] += 1
    assert owner.min() == 1 and owner.max() == 1


@pytest.mark.parametrize("nx,ny,nz", GRIDS)
def test_plane_issue_order_covers_what_the_warps_wait_for(nx, ny, nz):
    # issue order of a CTA's plane copies (plane t of every z group, t ascending, the two planes above a
    # group being planes 0, 1 of the next): every staged plane 0..zl+1 exactly once, and a group's own planes
    # in the order it marches through them
    g = P.brick_plan(nx, ny, nz, 148, SMEM)
    for zl in {g["zlen"], nz - (g["pz"] - 1) * g["zlen"]}:
        order = []
        for t in range(g["ppg"] + 2):
            for gi in range(g["ngrp"]):
                if t >= g["ppg"] and gi + 1 < g["ngrp"]:
                    continue
                s = gi * g["ppg"] + t
                if s <= zl + 1:
                    order.append(s)
        assert sorted(order) == list(range(zl + 2))
        pos = {s: i for i, s in enumerate(order)}
        for gi in range(g["ngrp"]):
            # (the two planes above a group are the next group's planes 0, 1: issued early, never late)
            need = [s for s in range(gi * g["ppg"], gi * g["ppg"] + g["ppg"]) if s <= zl + 1]
            assert [pos[s] for s in need] == sorted(pos[s] for s in need)


def test_no_plan_for_unsupported_grids():
    assert P.brick_plan(127, 64, 64) is None          # odd nx: 16-byte pairs straddle lines
    assert P.brick_plan(256, 64, 64) is None          # nx + 4 > 256 (tensor-map box limit)
    assert P.brick_plan(160, 160, 80) is None         # 83 % lane fill: > 8 planes per warp on 148 CTAs
    assert P.brick_plan(128, 200, 150) is None        # 3.8M rows exceed 148 x 32 warps x 8 planes x 64 points


def test_c4_plan():
    g = P.brick_plan(128, 128, 128, 148, SMEM)
    assert g["py"] * g["pz"] == 128 and g["ppg"] == 8 and g["ylen"] * g["zlen"] == 128
