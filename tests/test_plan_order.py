"""Entry order of the bank-permuted full-ring plans (gh_internal.cuh
order_lane_monotone, used by permute_for_banks for the c1/c2 plans), host-side.

The c1/c2 gather runs bank-permuted entries: entries (2k, 2k+1) must hold bins
with complementary row-parity vectors (no shared-memory bank conflict), and
the reference's tie rule (argmax_index keeps the first maximum,
src/direct.cpp:55-62) must survive the permutation: each of the gather's 8
lane groups (entry mod 8) meets its bins in increasing order in the ordered
part, so "first strict maximum" per lane is the smallest bin; the rest is an
ascending tail from `tie_from` on, which the gather flags on equality
(kernel 3). The header is compiled with g++ here: no GPU needed.
"""
import subprocess
import textwrap
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SRC = textwrap.dedent(r"""
    #include "paper_2307_16550_b200/csrc/gh_internal.cuh"
    #include <cstdio>
    #include <cstdlib>
    #include <vector>
    // args: n_bins P seed skew ; prints "ok <tie_from> <n>" or the first violation
    int main(int argc, char** argv) {
      const int n = atoi(argv[1]), P = atoi(argv[2]);
      uint64_t st = strtoull(argv[3], nullptr, 10);
      const int skew = atoi(argv[4]);  // per cent of bins forced into class 0
      const unsigned full = (1u << P) - 1u;
      std::vector<uint32_t> uniq;
      std::vector<unsigned> par;
      for (int b = 0; b < n; ++b) {
        st = gh::splitmix64(st);
        if (st % 97 == 0) continue;  // bins dropped as duplicates: uniq has gaps
        uniq.push_back((uint32_t)b);
        st = gh::splitmix64(st);
        par.push_back((int)(st % 100) < skew ? 0u : (unsigned)((st >> 8) & full));
      }
      std::vector<uint32_t> order;
      const int64_t tie = gh::order_lane_monotone(uniq, par, P, &order);
      if (order.size() != uniq.size()) { printf("size\n"); return 1; }
      if (tie % 32 != 0 || tie < 0 || tie > (int64_t)order.size()) { printf("tie_from %lld\n", (long long)tie); return 1; }
      std::vector<int> pos(n, -1), cls(n, -1);
      for (size_t i = 0; i < uniq.size(); ++i) cls[uniq[i]] = (int)par[i];
      for (size_t e = 0; e < order.size(); ++e) {
        if (order[e] >= (uint32_t)n || cls[order[e]] < 0 || pos[order[e]] >= 0) { printf("not a permutation at %zu\n", e); return 1; }
        pos[order[e]] = (int)e;
      }
      for (int64_t e = 0; e + 1 < tie; e += 2)
        if (((unsigned)cls[order[e]] ^ (unsigned)cls[order[e + 1]]) != full) { printf("pair %lld not complementary\n", (long long)e); return 1; }
      for (int64_t e = 8; e < tie; ++e)
        if (order[e] <= order[e - 8]) { printf("lane group order at %lld\n", (long long)e); return 1; }
      for (size_t e = (size_t)tie + 1; e < order.size(); ++e)
        if (order[e] <= order[e - 1]) { printf("tail order at %zu\n", e); return 1; }
      printf("ok %lld %zu\n", (long long)tie, order.size());
      return 0;
    }
""")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    d = tmp_path_factory.mktemp("plan_order")
    src = d / "check.cpp"
    src.write_text(SRC)
    exe = d / "check"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I/usr/local/cuda/include", f"-I{ROOT}",
                        "-x", "c++", str(src), "-o", str(exe)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("g++ / CUDA headers unavailable: " + r.stderr[-300:])
    return exe


@pytest.mark.parametrize("n,P,seed,skew", [
    (40000, 3, 1, 0),     # c1/c2: 200 x 200 bins, 3 pairs, balanced classes
    (40000, 3, 2, 20),    # one class over-represented: a long tail
    (5000, 2, 3, 0),      # two couples, two pair classes each
    (1000, 1, 4, 0),      # one couple over the four pair classes
    (37, 3, 5, 0),        # fewer bins than one block: everything in the tail
])
def test_ordered_plan_is_complementary_and_lane_monotone(checker, n, P, seed, skew):
    r = subprocess.run([str(checker), str(n), str(P), str(seed), str(skew)], capture_output=True,
                       text=True)
    out = r.stdout.split()
    assert out and out[0] == "ok", r.stdout + r.stderr
    tie_from, total = int(out[1]), int(out[2])
    if n >= 1000 and skew == 0:
        assert tie_from > 0.9 * total  # balanced classes: a short tail
