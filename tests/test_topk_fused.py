"""Map-free top-K local maxima — the gather with the prune test in its loop
(gh_gather_pick.cu k_gather_pick, engine "pick") and the halo-tile kernel
(gh_gather_topk.cu k_gather_topk, engine "fused") — against the
map-then-pick path (k_gather map mode + k_topk_localmax, the same fp32
values) and the fp64 oracle.

The fused pick must return exactly what the unfused path returns: the
same bins and bit-identical values (both sum the same staged powers in the
same pair order); the rule is the oracle's or_topk_local_max (a bin beats
smaller-index neighbours strictly and larger-index ones or ties; ranking by
value desc, bin asc; tie rule of src/direct.cpp:55-62).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2307_16550_b200 as gh
from paper_2307_16550_b200 import scene as S
from oracle import oracle as O

from test_gpu_parity import frames_to_dev, topk_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["pick", "fused"])
def fused_engine(ctx, request):
    # these tests pin the map-free engine; the session context is shared
    ctx.set_topk_impl(request.param)
    yield request.param
    ctx.set_topk_impl("auto")


def c3_sub(nx=240, ny=202):
    # BASELINE c3 stations / waveform (16 pairs, N = 1024, M = 4096) on a
    # sub-grid: a tiled table, so the fused plan applies
    c3 = S.baseline("c3")
    sp = c3.grid_spacing[0]
    ox, oy = -sp * (nx - 1) / 2, -sp * (ny - 1) / 2
    return c3.with_(grid_n=(nx, ny, 1), grid_origin=(ox, oy, 0.0),
                    area_lo=(ox - sp / 2, oy - sp / 2, 0.0),
                    area_hi=(-ox + sp / 2, -oy + sp / 2, 0.0))


def unfused(ctx, sc, table, fd, k):
    m = gh.hop_decision_map(ctx, table, fd)
    return gh.topk_local_max(ctx, sc, m, k)


@pytest.mark.parametrize("k", [1, 5, 8])
def test_fused_equals_map_then_pick(ctx, k):
    sc = c3_sub()
    T = 37  # not a multiple of the 8-trial batch
    t = gh.precompute_hop_table(ctx, sc)
    fr, _ = O.synth(sc, 11, T)
    fd = frames_to_dev(fr)
    fi, fv = gh.hop_topk(ctx, t, fd, k)
    ui, uv = unfused(ctx, sc, t, fd, k)
    assert np.array_equal(fi.cpu().numpy(), ui.cpu().numpy())
    assert np.array_equal(fv.cpu().numpy(), uv.cpu().numpy())
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    topk_parity(ref, fi.cpu().numpy(), sc, k, f"fused top-{k}")


def test_fused_zero_frames_plateau(ctx):
    # an all-zero map is one plateau: only its smallest bin is a local maximum
    sc = c3_sub(120, 98)
    t = gh.precompute_hop_table(ctx, sc)
    z = torch.zeros((9, sc.n_pairs, sc.n_samples), dtype=torch.complex64, device="cuda")
    fi, fv = gh.hop_topk(ctx, t, z, 4)
    fi = fi.cpu().numpy()
    assert (fi[:, 0] == 0).all() and (fi[:, 1:] == -1).all()
    assert (fv.cpu().numpy() == 0).all()


def test_fused_campaign_and_host_entry(ctx):
    sc = c3_sub()
    T, k = 24, 5
    t = gh.precompute_hop_table(ctx, sc)
    ci, cv = gh.campaign_hop_topk(ctx, t, sc, 100, T, k)
    fr, _ = O.synth(sc, 100, T)
    ui, uv = unfused(ctx, sc, t, frames_to_dev(fr), k)
    # synthesis on the device vs the oracle's frames: near-equal maps, so
    # compare against the oracle rule with the tie tolerance
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    topk_parity(ref, ci.cpu().numpy(), sc, k, "campaign fused")
    hi, hv = gh.api.hop_estimate_topk(ctx, t, fr, k)
    assert np.array_equal(hi, ui.cpu().numpy())
    assert np.allclose(hv, uv.cpu().numpy().astype(np.float64), rtol=0, atol=0)


def test_fused_c3_full_grid_vs_unfused(ctx):
    sc = S.baseline("c3")
    T, k = 19, 5
    t = gh.precompute_hop_table(ctx, sc)
    fr, _ = O.synth(sc, 7, T)
    fd = frames_to_dev(fr)
    fi, fv = gh.hop_topk(ctx, t, fd, k)
    ui, uv = unfused(ctx, sc, t, fd, k)
    assert np.array_equal(fi.cpu().numpy(), ui.cpu().numpy())
    assert np.array_equal(fv.cpu().numpy(), uv.cpu().numpy())


def test_topk_engines_agree_on_a_ragged_batch(ctx):
    # the 'map' engine through the same entry point: identical bins/values
    sc = c3_sub(130, 114)
    T, k = 13, 6
    t = gh.precompute_hop_table(ctx, sc)
    fr, _ = O.synth(sc, 3, T)
    fd = frames_to_dev(fr)
    fi, fv = gh.hop_topk(ctx, t, fd, k)
    ctx.set_topk_impl("map")
    mi, mv = gh.hop_topk(ctx, t, fd, k)
    assert np.array_equal(fi.cpu().numpy(), mi.cpu().numpy())
    assert np.array_equal(fv.cpu().numpy(), mv.cpu().numpy())


def test_pick_3d_grid_and_halo_shards(ctx, fused_engine):
    # the pick engine on a 3-D lattice (26 neighbours) and on halo shards
    # (core layers only, neighbours inside the shard's layers): identical to
    # the map engine through the same entry point
    if fused_engine != "pick":
        pytest.skip("the halo-tile kernel is 2-D only")
    from test_gpu_parity import c5_reduced
    c5 = c5_reduced()
    sc = c5.with_(tx=c5.tx[:12], rx=c5.rx[:12])  # 12 pairs: a tiled plan the engine takes
    T, k = 21, 3
    fr, _ = O.synth(sc, 9, T)
    fd = frames_to_dev(fr)
    tables = [gh.precompute_hop_table(ctx, sc),
              gh.precompute_hop_table_shard(ctx, sc, 2, 5, halo=True),
              gh.precompute_hop_table_shard(ctx, sc, 0, 3, halo=False)]
    for t in tables:
        ctx.set_topk_impl("pick")
        pi, pv = gh.hop_topk(ctx, t, fd, k)
        ctx.set_topk_impl("map")
        mi, mv = gh.hop_topk(ctx, t, fd, k)
        assert np.array_equal(pi.cpu().numpy(), mi.cpu().numpy())
        assert np.array_equal(pv.cpu().numpy(), mv.cpu().numpy())
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    ctx.set_topk_impl("pick")
    pi, _ = gh.hop_topk(ctx, tables[0], fd, k)
    topk_parity(ref, pi.cpu().numpy(), sc, k, "pick 3-D")


def test_auto_engine_takes_pick_on_large_batches(ctx, fused_engine):
    # auto: >= one 8-trial batch per SM -> the pick engine; same lists as map
    if fused_engine != "pick":
        pytest.skip("engine-independent")
    sc = c3_sub(96, 82)
    T, k = 8 * 148 * 2 - 3, 5  # two full rounds of one batch per SM, the last batch ragged
    t = gh.precompute_hop_table(ctx, sc)
    ctx.set_topk_impl("auto")
    ai, av = gh.campaign_hop_topk(ctx, t, sc, 0, T, k)
    ctx.set_topk_impl("map")
    mi, mv = gh.campaign_hop_topk(ctx, t, sc, 0, T, k)
    assert np.array_equal(ai.cpu().numpy(), mi.cpu().numpy())
    assert np.array_equal(av.cpu().numpy(), mv.cpu().numpy())


def test_pick_engine_bounds_checked_build(ctx, fused_engine):
    # compute-sanitizer's stand-in: the CHECK instantiation of k_gather_pick
    # tests every staged shared-memory offset, window extent, queue slot and
    # table / spectra row; it must run clean and return the same lists
    if fused_engine != "pick":
        pytest.skip("the bounds-tested build belongs to the pick engine")
    for sc, T, k in ((c3_sub(), 37, 5), (c3_sub(120, 98), 9, 4), (S.baseline("c3"), 19, 5)):
        t = gh.precompute_hop_table(ctx, sc)
        fr, _ = O.synth(sc, 21, T)
        fd = frames_to_dev(fr)
        pi, pv = gh.hop_topk(ctx, t, fd, k)
        ctx.set_debug_checks(True)
        try:
            ci, cv = gh.hop_topk(ctx, t, fd, k)
            zi, _ = gh.hop_topk(ctx, t, torch.zeros_like(fd), k)  # every bin a candidate
        finally:
            ctx.set_debug_checks(False)
        assert np.array_equal(ci.cpu().numpy(), pi.cpu().numpy())
        assert np.array_equal(cv.cpu().numpy(), pv.cpu().numpy())
        assert (zi.cpu().numpy()[:, 0] == 0).all()


def test_argmax_through_the_pick_engine(ctx, fused_engine):
    # hop_argmax with at least one 8-trial batch per SM on a tiled K = 1 plan
    # runs the pick engine's K = 1 form: the same bins and values as the
    # plain fused-argmax gather (small batches) and as the maps' first maximum
    if fused_engine != "pick":
        pytest.skip("engine-independent")
    ctx.set_topk_impl("auto")
    sc = c3_sub(96, 82)
    T = 8 * 148 * 2 - 3  # two full rounds of one batch per SM, the last batch ragged
    t = gh.precompute_hop_table(ctx, sc)
    fr, _ = gh.synthesize(ctx, sc, 0, T)
    bi, bv = gh.hop_argmax(ctx, t, fr)                       # routed: 296 batches
    parts = [gh.hop_argmax(ctx, t, fr[a:a + 512]) for a in range(0, T, 512)]  # plain gather
    pi = torch.cat([p[0] for p in parts])
    pv = torch.cat([p[1] for p in parts])
    assert np.array_equal(bi.cpu().numpy(), pi.cpu().numpy())
    assert np.array_equal(bv.cpu().numpy(), pv.cpu().numpy())
    m = gh.hop_decision_map(ctx, t, fr[:64]).cpu().numpy()
    assert np.array_equal(bi.cpu().numpy()[:64], m.argmax(axis=1))
    # zero frames: the plateau's first bin
    zi, zv = gh.hop_argmax(ctx, t, torch.zeros_like(fr))
    assert (zi.cpu().numpy() == 0).all() and (zv.cpu().numpy() == 0).all()
