"""Tile entry order of the gather plans (gh_internal.cuh tile_local), host-side.

The tiled argmax plans order a tile's entries in 8-bin blocks (2 x 4 x 1 on
2-D grids, 2 x 1 x 4 on 3-D ones) so a half-warp of the gather reads a
compact patch. Two properties carry the parity argument (k_gather):
the order is a bijection onto the tile box, and every gather lane (entries
lb = 16 s + sub, sub < 16, of a warp run starting at a multiple of 16) meets
its bins in increasing global order, so "first strict maximum" per lane plus
smallest-bin merges keeps the reference's tie rule (direct.cpp:55-62).
The header is compiled with g++ here: no GPU needed.
"""
import subprocess
import textwrap
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SRC = textwrap.dedent(r"""
    #include "paper_2307_16550_b200/csrc/gh_internal.cuh"
    #include <cstdio>
    #include <vector>
    // args: wx wy wz blk ; prints "ok" or the first violation
    int main(int argc, char** argv) {
      gh::TileDesc td{};
      td.wx = atoi(argv[1]); td.wy = atoi(argv[2]); td.wz = atoi(argv[3]); td.blk = atoi(argv[4]);
      const int64_t nb = (int64_t)td.wx * td.wy * td.wz;
      const int64_t nx = 1000, ny = 1000;  // an enclosing lattice
      std::vector<int> seen(nb, 0);
      std::vector<int64_t> gb(nb);
      for (int64_t lb = 0; lb < nb; ++lb) {
        int64_t x, y, z;
        gh::tile_local(td, lb, &x, &y, &z);
        if (x < 0 || x >= td.wx || y < 0 || y >= td.wy || z < 0 || z >= td.wz) {
          printf("out of box lb=%lld\n", (long long)lb); return 1;
        }
        const int64_t k = (z * td.wy + y) * td.wx + x;
        if (seen[k]++) { printf("duplicate lb=%lld\n", (long long)lb); return 1; }
        gb[lb] = x + nx * (y + ny * z);
      }
      for (int sub = 0; sub < 16; ++sub)
        for (int64_t lb = sub + 16; lb < nb; lb += 16)
          if (gb[lb] <= gb[lb - 16]) { printf("lane order lb=%lld\n", (long long)lb); return 1; }
      printf("ok\n");
      return 0;
    }
""")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    d = tmp_path_factory.mktemp("tile_order")
    src = d / "check.cpp"
    src.write_text(SRC)
    exe = d / "check"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I/usr/local/cuda/include", f"-I{ROOT}",
                        "-x", "c++", str(src), "-o", str(exe)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("g++ / CUDA headers unavailable: " + r.stderr[-300:])
    return exe


def blk_code(sx, sy, sz):
    return 1 + sx + (sy << 2) + (sz << 4)


@pytest.mark.parametrize("dims,blk", [
    ((112, 112, 1), blk_code(1, 2, 0)),   # c3-like 2-D tile, 2 x 4 x 1 blocks
    ((8, 4, 1), blk_code(1, 2, 0)),
    ((32, 24, 8), blk_code(1, 0, 2)),     # 3-D tile, 2 x 1 x 4 blocks
    ((64, 64, 4), blk_code(1, 0, 2)),
    ((113, 57, 1), 0),                    # ragged edge tile: plain order
    ((10, 6, 3), 0),
])
def test_tile_local_bijective_and_lane_monotone(checker, dims, blk):
    r = subprocess.run([str(checker), *map(str, dims), str(blk)], capture_output=True, text=True)
    assert r.stdout.strip() == "ok", r.stdout + r.stderr
