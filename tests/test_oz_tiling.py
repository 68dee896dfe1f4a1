"""Host restatement of the INT8 V path's tile bookkeeping (csrc/pair_oz.cu OzWalk / oz_tiles,
pair_kr.cu's 16 x 8 tile numbering), checked on CPU: every walker pair q > p of an ensemble is
covered exactly once by the V-GEMM tiles (16 Q walkers x 8 or 10 P walkers), the persistent
CTAs' strided walks visit each tile once, and the o-tile addresses the fused epilogue reads
stay inside the o buffer written by pair_kr_kernel<false, 2> (all that are read are in range;
pairs past the triangle row are masked on the device)."""
import pytest


def row_len(a, pw):
    return (16 * (a + 1) + pw - 1) // pw


def oz_tiles(nbq, pw):
    return sum(row_len(a, pw) for a in range(nbq))


def walk(t0, stride, count, pw):  # OzWalk: settle() after the start and after every next()
    a, b = 0, t0
    out = []
    for _ in range(count):
        while b >= row_len(a, pw):
            b -= row_len(a, pw)
            a += 1
        out.append((a, b))
        b += stride
    return out


@pytest.mark.parametrize("m,pw", [(192, 10), (200, 10), (2048, 10), (512, 8), (2048, 8), (8192, 10)])
def test_tiles_cover_each_pair_once(m, pw):
    nbq = (m + 15) // 16
    ntiles = oz_tiles(nbq, pw)
    if pw == 8:
        assert ntiles == nbq * (nbq + 1)  # pair_kr's numbering t = a (a + 1) + b
    grid = min(148, ntiles)
    seen, tiles = {}, set()
    for cta in range(grid):
        my = (ntiles - 1 - cta) // grid + 1 if cta < ntiles else 0
        for it, (a, b) in enumerate(walk(cta, grid, my, pw)):
            t = cta + it * grid
            assert (a, b) not in tiles and t not in seen
            seen[t] = (a, b)
            tiles.add((a, b))
    assert sorted(seen) == list(range(ntiles))
    if m > 600:  # the pair-count check is O(m^2): the structural checks above suffice there
        return
    cover = {}
    for a, b in seen.values():
        for q in range(16 * a, 16 * a + 16):
            for p in range(pw * b, pw * b + pw):
                if q < m and p < m and q > p:
                    cover[(q, p)] = cover.get((q, p), 0) + 1
                    # the fused epilogue reads o of (q, p) in pair_kr tile a (a + 1) + p // 8
                    assert p < 16 * (a + 1)
                    assert a * (a + 1) + p // 8 < nbq * (nbq + 1)
    assert len(cover) == m * (m - 1) // 2 and set(cover.values()) == {1}
