"""GPU parity: the sm_100a path through the C ABI against the fp64 oracle.

Gates (BASELINE.json north_star):
  * location-bin indices identical to the oracle on every trial except
    documented near-ties (oracle top-2 within 1e-5 relative);
  * maps within 1e-4 relative: max|gpu - oracle| / max|oracle| per trial;
  * table indices bit-identical, coefficients within 1e-9.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2307_16550_b200 as gh
from paper_2307_16550_b200 import scene as S
from oracle import oracle as O

pytestmark = pytest.mark.gpu

MAP_TOL = 1e-4
TIE_TOL = 1e-5


def near_tie(m: np.ndarray, a: int, b: int) -> bool:
    top = m.max()
    return abs(m[a] - m[b]) <= TIE_TOL * abs(top)


def assert_argmax_parity(ref_maps, idx_gpu, what=""):
    bad = []
    for t, m in enumerate(ref_maps):
        a = int(np.argmax(m))
        g = int(idx_gpu[t])
        if a != g and not near_tie(m, a, g):
            bad.append((t, a, g, m[a], m[g]))
    assert not bad, f"{what}: {len(bad)} argmax mismatches (not near-ties): {bad[:5]}"


def rel_map_err(gpu, ref):
    err = np.abs(gpu.astype(np.float64) - ref).max(axis=1)
    return (err / np.abs(ref).max(axis=1)).max()


def frames_to_dev(fr):
    return torch.from_numpy(fr.astype(np.complex64)).cuda().contiguous()


@pytest.fixture(scope="module")
def small_scene():
    return S.small()


def test_table_indices_bit_identical(ctx):
    for scheme in (S.NEAREST, S.LINEAR, S.POLY3, S.POLAR):
        sc = S.small(scheme=scheme, nx=17, ny=13)
        t = gh.precompute_hop_table(ctx, sc)
        gi, gc = t.download()
        oi, oc, omr = O.build_table(sc)
        assert np.array_equal(gi, oi), f"scheme {scheme}: indices differ"
        assert np.abs(gc - oc).max() < 1e-9, f"scheme {scheme}: coefficients differ"
        assert abs(t.max_residual - omr) <= 1e-9 * max(1.0, omr)


def test_table_indices_baseline_c1(ctx):
    sc = S.baseline("c1")
    t = gh.precompute_hop_table(ctx, sc)
    gi, _ = t.download()
    oi, _, _ = O.build_table(sc)
    assert np.array_equal(gi, oi)


def test_table_window_error_names_bins(ctx):
    sc = S.small(wrap=False, bandwidth=1e9)  # aliases: ranges leave [0, N)
    with pytest.raises(gh.GridhopRuntimeError) as e:
        gh.precompute_hop_table(ctx, sc)
    assert "(bin" in str(e.value) and "hop table: sensed range outside" in str(e.value)
    with pytest.raises(O.OracleError) as eo:
        O.build_table(sc)
    assert str(e.value) == str(eo.value)


def test_synth_matches_oracle(ctx, small_scene):
    sc = small_scene
    fr_g, tr_g = gh.synthesize(ctx, sc, 5, 9)
    fr_o, tr_o = O.synth(sc, 5, 9)
    assert np.array_equal(tr_g.cpu().numpy(), tr_o)
    assert np.abs(fr_g.cpu().numpy() - fr_o).max() < 2e-5 * np.abs(fr_o).max()


@pytest.mark.parametrize("N,os", [(64, 4), (256, 4), (512, 2), (1024, 4), (128, 1)])
def test_spectra_match_oracle(ctx, N, os):
    rng = np.random.default_rng(N + os)
    fr = (rng.standard_normal((5, 3, N)) + 1j * rng.standard_normal((5, 3, N)))
    sp_g = gh.fast_time_spectra(ctx, frames_to_dev(fr), os).cpu().numpy()
    sp_o = O.spectra(fr, N * os)
    assert np.abs(sp_g - sp_o).max() < 1e-5 * np.abs(sp_o).max()


@pytest.mark.parametrize("scheme", [S.NEAREST, S.LINEAR, S.POLY3, S.POLAR])
@pytest.mark.parametrize("combine", [S.POWER, S.MAGNITUDE])
def test_hop_map_and_argmax(ctx, scheme, combine):
    sc = S.small(scheme=scheme)
    T = 37  # not a multiple of the 16/32-trial batch
    fr, _ = O.synth(sc, 0, T)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc, magnitude=combine == S.MAGNITUDE)
    t = gh.precompute_hop_table(ctx, sc)
    fd = frames_to_dev(fr)
    m = gh.hop_decision_map(ctx, t, fd, combine).cpu().numpy()
    assert rel_map_err(m, ref) < MAP_TOL
    idx, val = gh.hop_argmax(ctx, t, fd, combine)
    assert_argmax_parity(ref, idx.cpu().numpy(), f"scheme {scheme}")
    iv = idx.cpu().numpy()
    assert np.allclose(val.cpu().numpy(), ref[np.arange(T), iv], rtol=1e-4)


@pytest.mark.parametrize("os_", [4, 2])
@pytest.mark.parametrize("combine", [S.POWER, S.MAGNITUDE])
def test_hop_c1_scene_n256(ctx, os_, combine):
    # the c1/c2 scene (N = 256): the warp-resident two-stage FFT (k_fft256)
    # feeding the full-ring gather; T not a multiple of the 4-trial group
    sc = S.baseline("c1")
    if os_ != sc.os_range:
        sc = S.small(P=3, N=256, os=os_, nx=40, ny=30, scheme=S.NEAREST)
    T = 45
    fr, _ = O.synth(sc, 7, T)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc, magnitude=combine == S.MAGNITUDE)
    t = gh.precompute_hop_table(ctx, sc)
    fd = frames_to_dev(fr)
    m = gh.hop_decision_map(ctx, t, fd, combine).cpu().numpy()
    assert rel_map_err(m, ref) < MAP_TOL
    idx, _ = gh.hop_argmax(ctx, t, fd, combine)
    assert_argmax_parity(ref, idx.cpu().numpy(), f"c1 scene os={os_}")


def test_hop_tiled_plan_k1(ctx):
    # a scene whose full ring does not fit shared memory -> tiled plan
    sc = S.small(P=12, N=512, os=4, nx=60, ny=50, scheme=S.NEAREST)
    T = 40
    fr, _ = O.synth(sc, 0, T)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    t = gh.precompute_hop_table(ctx, sc)
    fd = frames_to_dev(fr)
    m = gh.hop_decision_map(ctx, t, fd).cpu().numpy()
    assert rel_map_err(m, ref) < MAP_TOL
    idx, _ = gh.hop_argmax(ctx, t, fd)
    assert_argmax_parity(ref, idx.cpu().numpy(), "tiled K=1")


def test_hop_estimate_host_buffers(ctx, small_scene):
    sc = small_scene
    fr, _ = O.synth(sc, 100, 21)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    t = gh.precompute_hop_table(ctx, sc)
    idx, val = gh.hop_estimate(ctx, t, fr)
    assert_argmax_parity(ref, idx, "host hop_estimate")
    with pytest.raises(gh.InvalidArgument, match="hop: frame shape mismatch"):
        gh.hop_estimate(ctx, t, fr[:, :2])


def test_hop_estimate_pipelined_chunks(ctx, small_scene):
    # >= 1024 trials: the host entry point pipelines H2D copies of ragged
    # trial chunks over two streams; results must equal the device path
    sc = small_scene
    T = 1029
    fr, _ = O.synth(sc, 7, T)
    t = gh.precompute_hop_table(ctx, sc)
    idx, val = gh.hop_estimate(ctx, t, fr)
    d_idx, d_val = gh.hop_argmax(ctx, t, frames_to_dev(fr))
    assert np.array_equal(idx, d_idx.cpu().numpy())
    assert np.array_equal(val, d_val.cpu().numpy().astype(np.float64))
    # and a second call reusing the context's buffers and events
    idx2, _ = gh.hop_estimate(ctx, t, fr[:1030 - 6])
    assert np.array_equal(idx2, idx[:1024])


def test_campaign_matches_oracle_campaign(ctx):
    sc = S.baseline("c1")
    T = 64
    oi, oc, _ = O.build_table(sc)
    o_idx, o_val = O.campaign_hop(sc, oi, oc, 0, T)
    t = gh.precompute_hop_table(ctx, sc)
    g_idx, g_val = gh.campaign_hop(ctx, t, sc, 0, T)
    g_idx = g_idx.cpu().numpy()
    fr, _ = O.synth(sc, 0, T)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    assert_argmax_parity(ref, g_idx, "c1 campaign")
    assert np.array_equal(np.argmax(ref, axis=1), o_idx)
    assert np.allclose(g_val.cpu().numpy(), o_val, rtol=1e-4)


@pytest.mark.parametrize("impl", ["tcgen05", "tcgen05_tf32", "tcgen05_v1", "simt"])
@pytest.mark.parametrize("combine", [S.POWER, S.MAGNITUDE])
def test_direct_map_and_argmax(ctx, combine, impl):
    sc = S.small()
    T = 19
    fr, _ = O.synth(sc, 3, T)
    ref = O.direct_map(sc, fr, magnitude=combine == S.MAGNITUDE)
    fd = frames_to_dev(fr)
    ctx.set_direct_impl(impl)
    try:
        m = gh.location_decision_map(ctx, sc, fd, combine).cpu().numpy()
        assert rel_map_err(m, ref) < MAP_TOL
        idx, _ = gh.direct_argmax(ctx, sc, fd, combine)
        assert_argmax_parity(ref, idx.cpu().numpy(), f"direct {impl}")
    finally:
        ctx.set_direct_impl("tcgen05")


@pytest.mark.parametrize("gain", [3.7e4, 2.5e-5])
def test_direct_fp16_frame_scaling(ctx, gain):
    # 3xFP16 scales frames by a power of two into [1, 2) before the fp16
    # split (fp16 max 65504, subnormals below 6e-5) and undoes it exactly
    sc = S.small()
    fr, _ = O.synth(sc, 11, 9)
    fr = fr * gain
    ref = O.direct_map(sc, fr)
    fd = frames_to_dev(fr)
    m = gh.location_decision_map(ctx, sc, fd).cpu().numpy()
    assert rel_map_err(m, ref) < MAP_TOL
    idx, _ = gh.direct_argmax(ctx, sc, fd)
    assert_argmax_parity(ref, idx.cpu().numpy(), f"direct fp16 x{gain}")


def test_direct_fp16_mixed_trial_amplitudes(ctx):
    # every trial is scaled by its own power of two: a batch mixing trials
    # 9 decades apart keeps each trial's map as accurate as on its own (one
    # batch-wide exponent would push the weak trials' fp16 parts into
    # subnormals)
    sc = S.small()
    T = 12
    fr, _ = O.synth(sc, 5, T)
    gains = np.array([1e4, 1e-5, 1.0, 3e-3] * 3)[:, None, None]
    fr = fr * gains
    ref = O.direct_map(sc, fr)
    fd = frames_to_dev(fr)
    m = gh.location_decision_map(ctx, sc, fd).cpu().numpy()
    for t in range(T):
        assert rel_map_err(m[t:t + 1], ref[t:t + 1]) < MAP_TOL, t
    idx, _ = gh.direct_argmax(ctx, sc, fd)
    assert_argmax_parity(ref, idx.cpu().numpy(), "direct fp16 mixed amplitudes")


def test_direct_fast_mode_parity_loss(ctx):
    # the 1xFP16 fast mode (one MMA per K step): a third
    # of the tensor work. Its operands carry 11-bit mantissas, so single
    # products are off by ~5e-4; over N = 256 samples the map error against
    # the map maximum comes out just under the 1e-4 bar on c2 (measured
    # 7.8e-5, the 3xFP16 default: ~1e-6) — too close to be the default. The
    # loss is bounded and printed here.
    sc = S.baseline("c2")
    T = 64
    fr, _ = O.synth(sc, 0, T)
    sub = np.arange(0, T, 8)
    ref = O.direct_map(sc, fr[sub])
    fd = frames_to_dev(fr)
    exact = gh.location_decision_map(ctx, sc, fd).cpu().numpy()[sub]
    ctx.set_direct_impl("tcgen05_fast")
    try:
        fast = gh.location_decision_map(ctx, sc, fd).cpu().numpy()[sub]
        fidx, _ = gh.direct_argmax(ctx, sc, fd)
    finally:
        ctx.set_direct_impl("tcgen05")
    e_exact, e_fast = rel_map_err(exact, ref), rel_map_err(fast, ref)
    assert e_exact < MAP_TOL
    assert 10 * e_exact < e_fast < 5e-4, (e_exact, e_fast)
    agree = np.mean(fidx.cpu().numpy()[sub] == ref.argmax(axis=1))
    assert agree >= 0.75, agree
    print(f"1xFP16 fast mode: map error {e_fast:.2e} (3xFP16 {e_exact:.2e}), argmax agreement {agree:.2f}")


def test_direct_tcgen05_c2_scale(ctx):
    # the c2 scene (40,000 bins x 3 pairs, N = 256), 130 trials: two trial
    # tiles of 128 (ragged) through the tensor-core path
    sc = S.baseline("c2")
    T = 130
    fr, _ = O.synth(sc, 0, T)
    sub = np.arange(0, T, 13)
    ref = O.direct_map(sc, fr[sub])
    fd = frames_to_dev(fr)
    m = gh.location_decision_map(ctx, sc, fd).cpu().numpy()
    assert rel_map_err(m[sub], ref) < MAP_TOL
    idx, _ = gh.direct_argmax(ctx, sc, fd)
    assert_argmax_parity(ref, idx.cpu().numpy()[sub], "direct c2")
    # per-element relative error on the peak neighbourhood (3xTF32 ~ fp32)
    peak = ref.max(axis=1, keepdims=True)
    big = ref > 0.1 * peak
    assert (np.abs(m[sub] - ref)[big] / ref[big]).max() < 1e-4


def test_edge_cases(ctx, small_scene):
    sc = small_scene
    t = gh.precompute_hop_table(ctx, sc)
    empty = torch.empty((0, sc.n_pairs, sc.n_samples), dtype=torch.complex64, device="cuda")
    idx, val = gh.hop_argmax(ctx, t, empty)
    assert idx.numel() == 0
    with pytest.raises(gh.InvalidArgument, match="unknown interpolation scheme"):
        gh.precompute_hop_table(ctx, sc, scheme=9)
    with pytest.raises(gh.InvalidArgument, match="empty grid"):
        gh.precompute_hop_table(ctx, sc.with_(grid_n=(0, 4, 1)))
    # single trial
    fr, _ = O.synth(sc, 0, 1)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    idx, _ = gh.hop_argmax(ctx, t, frames_to_dev(fr))
    assert_argmax_parity(ref, idx.cpu().numpy(), "T=1")


def topk_parity(ref_maps, gidx, sc, k, what):
    bad = []
    for t, m in enumerate(ref_maps):
        oi, ov = O.topk_local_max(sc, m, k)
        gi = gidx[t]
        for j in range(k):
            if oi[j] == gi[j]:
                continue
            # allowed only when the two candidates are a near-tie in value
            a = m[oi[j]] if oi[j] >= 0 else 0.0
            b = m[gi[j]] if gi[j] >= 0 else 0.0
            if abs(a - b) > TIE_TOL * m.max():
                bad.append((t, j, oi[j], gi[j], a, b))
    assert not bad, f"{what}: top-k mismatches {bad[:4]}"


def test_hop_topk_multi_target(ctx):
    sc = S.small(n_targets=3, amp_mode=S.AMP_CGAUSS_PER_PAIR, snr_mode=S.SNR_UNIFORM_PER_PAIR,
                 snr_lo=5.0, snr_hi=20.0, nx=30, ny=26, scheme=S.NEAREST)
    T, K = 21, 3
    fr, _ = O.synth(sc, 0, T)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    t = gh.precompute_hop_table(ctx, sc)
    gidx, gval = gh.hop_topk(ctx, t, frames_to_dev(fr), K)
    topk_parity(ref, gidx.cpu().numpy(), sc, K, "small top-3")
    # campaign form (synthesis on the device) picks the same peaks
    cidx, _ = gh.campaign_hop_topk(ctx, t, sc, 0, T, K)
    topk_parity(ref, cidx.cpu().numpy(), sc, K, "campaign top-3")
    # the same kernel on caller maps
    m = gh.hop_decision_map(ctx, t, frames_to_dev(fr))
    midx, _ = gh.topk_local_max(ctx, sc, m, K)
    topk_parity(ref, midx.cpu().numpy(), sc, K, "maps top-3")


def test_c3_full_grid_top5(ctx):
    # BASELINE c3 at full size: 10^6 bins, 16 pairs, N = 1024, M = 4096,
    # tiled 32-trial plan; a few trials against the oracle
    sc = S.baseline("c3")
    T, K = 6, 5
    t = gh.precompute_hop_table(ctx, sc)
    gi_, _ = t.download()
    oi, oc, _ = O.build_table(sc)
    assert np.array_equal(gi_, oi)
    fr, truth = O.synth(sc, 0, T)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    gidx, _ = gh.hop_topk(ctx, t, frames_to_dev(fr), K)
    topk_parity(ref, gidx.cpu().numpy(), sc, K, "c3 top-5")
    cidx, _ = gh.campaign_hop_topk(ctx, t, sc, 0, T, K)
    topk_parity(ref, cidx.cpu().numpy(), sc, K, "c3 campaign top-5")


@pytest.mark.parametrize("scheme", [S.POLY3, S.POLAR])
def test_c4_geometry_tiled_complex(ctx, scheme):
    # c4 stations/waveform (16 pairs, N = 512, os = 2, K = 3) on a 160 x 160
    # sub-grid: the tiled complex-spectrum plan at realistic tile sizes
    c4 = S.baseline("c4")
    sc = c4.with_(grid_n=(160, 160, 1), grid_origin=(-15.9, -15.9, 0.0), scheme=scheme,
                  area_lo=(-16.0, -16.0, 0.0), area_hi=(16.0, 16.0, 0.0))
    T = 33
    oi, oc, _ = O.build_table(sc)
    t = gh.precompute_hop_table(ctx, sc)
    gi_, gc_ = t.download()
    assert np.array_equal(gi_, oi) and np.abs(gc_ - oc).max() < 1e-9
    fr, _ = O.synth(sc, 0, T, snr_db=0.0)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    fd = frames_to_dev(fr)
    m = gh.hop_decision_map(ctx, t, fd).cpu().numpy()
    assert rel_map_err(m, ref) < MAP_TOL
    idx, _ = gh.campaign_hop(ctx, t, sc, 0, T, snr_db=0.0)
    assert_argmax_parity(ref, idx.cpu().numpy(), f"c4 scheme {scheme}")


def test_campaign_statistics_match_oracle(ctx):
    # RMSE / hit-ratio curve points (c1 scene, 3 SNRs): identical estimates
    # give identical statistics
    from paper_2307_16550_b200 import distributed as D
    sc = S.baseline("c1")
    T = 96
    oi, oc, _ = O.build_table(sc)
    t = gh.precompute_hop_table(ctx, sc)
    for snr in (0.0, 10.0, 20.0):
        o_idx, _ = O.campaign_hop(sc, oi, oc, 0, T, snr_db=snr)
        g_idx, _ = gh.campaign_hop(ctx, t, sc, 0, T, snr_db=snr)
        _, truth = O.synth(sc, 0, T, snr_db=snr)
        so = D.campaign_stats(sc, o_idx, truth)
        sg = D.campaign_stats(sc, g_idx.cpu().numpy(), truth)
        assert np.allclose(so, sg), (snr, so, sg)


@pytest.mark.parametrize("P,scheme,combine,T", [
    (64, S.NEAREST, S.POWER, 1500),  # compile-time 64 pairs, many items per CTA
    (20, S.POLY3, S.MAGNITUDE, 700),  # runtime pair count, a partial last chunk
    (40, S.NEAREST, S.MAGNITUDE, 333),
])
def test_pipelined_tiled_gather(ctx, P, scheme, combine, T):
    # > 16 pairs: the persistent gather whose producer warp restages pair
    # chunks of the next (tile, batch) item under the current one; enough
    # trials that every CTA runs several items (phase flips, ring reuse)
    sc = S.small(P=P, N=512, os=4, nx=40, ny=36, scheme=scheme)
    fr, _ = O.synth(sc, 0, T)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc, magnitude=combine == S.MAGNITUDE)
    t = gh.precompute_hop_table(ctx, sc)
    fd = frames_to_dev(fr)
    idx, val = gh.hop_argmax(ctx, t, fd, combine)
    assert_argmax_parity(ref, idx.cpu().numpy(), f"P={P}")
    iv = idx.cpu().numpy()
    assert np.allclose(val.cpu().numpy(), ref[np.arange(T), iv], rtol=1e-4)
    m = gh.hop_decision_map(ctx, t, fd[:97], combine).cpu().numpy()
    assert rel_map_err(m, ref[:97]) < MAP_TOL
    # repeated launches agree bit for bit (no stale chunk is ever read)
    idx2, val2 = gh.hop_argmax(ctx, t, fd, combine)
    assert torch.equal(idx, idx2) and torch.equal(val, val2)


def test_blocked_plan_exact_ties_smallest_bin(ctx):
    # a tiled 8-trial plan (12 pairs, N = 512) whose entries run in 2 x 4
    # blocks, on a grid fine enough that neighbouring bins share every
    # pair's range row: their sums are bit-identical, and the argmax must
    # still return the smallest bin of a tied maximum (direct.cpp:55-62)
    nx, ny, sp = 60, 48, 0.08
    ox, oy = -sp * (nx - 1) / 2, -sp * (ny - 1) / 2
    sc = S.small(P=12, N=512, os=4, nx=nx, ny=ny, scheme=S.NEAREST).with_(
        grid_spacing=(sp, sp, 1.0), grid_origin=(ox, oy, 0.0),
        area_lo=(ox - sp / 2, oy - sp / 2, 0.0), area_hi=(-ox + sp / 2, -oy + sp / 2, 0.0))
    T = 64
    fr, _ = O.synth(sc, 3, T)
    oi, oc, _ = O.build_table(sc)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    t = gh.precompute_hop_table(ctx, sc)
    idx = gh.hop_argmax(ctx, t, frames_to_dev(fr))[0].cpu().numpy()
    assert_argmax_parity(ref, idx, "blocked plan")
    m = gh.hop_decision_map(ctx, t, frames_to_dev(fr)).cpu().numpy()
    ties = 0
    for k in range(T):
        top = np.flatnonzero(m[k] == m[k].max())  # exact ties on the device map
        if len(top) > 1:
            ties += 1
            assert idx[k] == top[0], (k, idx[k], top[:4])
    assert ties > 0, "scene produced no exact ties"


def c5_reduced():
    # BASELINE c5 stations/waveform (64 pairs, N = 512, os = 4, 3-D grid
    # spacing 0.195 x 0.195 x 0.3125 m) on a 48 x 40 x 8 block of the grid
    c5 = S.baseline("c5")
    sx, sz = c5.grid_spacing[0], c5.grid_spacing[2]
    return c5.with_(grid_n=(48, 40, 8), grid_origin=(-4.7, -3.9, 8.0 + sz / 2),
                    area_lo=(-4.8, -4.0, 8.0), area_hi=(-4.8 + 48 * sx, -4.0 + 40 * sx, 8.0 + 8 * sz))


def test_c5_geometry_3d_and_grid_sharding(ctx):
    from paper_2307_16550_b200 import distributed as D
    sc = c5_reduced()
    T = 24
    oi, oc, _ = O.build_table(sc)
    full = gh.precompute_hop_table(ctx, sc)
    gi_, _ = full.download()
    assert np.array_equal(gi_, oi)
    fr, _ = O.synth(sc, 0, T)
    ref = O.hop_map(O.spectra(fr, sc.n_fft), oi, oc)
    fd = frames_to_dev(fr)
    m = gh.hop_decision_map(ctx, full, fd).cpu().numpy()
    assert rel_map_err(m, ref) < MAP_TOL
    g_idx, _ = gh.hop_argmax(ctx, full, fd)
    assert_argmax_parity(ref, g_idx.cpu().numpy(), "c5 reduced")
    # two location-grid shards (z layers 0-3 and 3-8): shard rows equal the
    # full table, and merging shard winners by key == the full argmax
    keys = np.zeros(T, dtype=np.int64)
    for lo, hi in ((0, 3), (3, 8)):
        sh = gh.precompute_hop_table_shard(ctx, sc, lo, hi)
        b0, b1 = sc.slab_bins(lo, hi)
        si, _ = sh.download()
        assert np.array_equal(si, oi[b0:b1])
        sm_ = gh.hop_decision_map(ctx, sh, fd).cpu().numpy()
        assert np.abs(sm_ - m[:, b0:b1]).max() <= 1e-6 * np.abs(m).max()
        ix, vx = gh.hop_argmax(ctx, sh, fd)
        keys = np.maximum(keys, D.encode_keys(vx.cpu().numpy(), ix.cpu().numpy()))
    bins, _ = D.decode_keys(keys)
    assert np.array_equal(bins, g_idx.cpu().numpy())


@pytest.mark.parametrize("name", ["small", "c2"])
def test_full_ring_exact_ties_smallest_bin(ctx, name):
    # Full-ring plans (c1/c2-like, P <= 8) run bank-permuted entries, so
    # entry order is not bin order. Exact ties must still resolve to the
    # smallest bin (argmax_index, src/direct.cpp:55-62): all-zero frames tie
    # every bin at 0 -> bin 0; a mirror-symmetric scene ties mirrored bins.
    sc = S.small() if name == "small" else S.baseline("c2")
    t = gh.precompute_hop_table(ctx, sc)
    T = 40
    zero = torch.zeros((T, sc.n_pairs, sc.n_samples), dtype=torch.complex64, device="cuda")
    idx, val = gh.hop_argmax(ctx, t, zero)
    assert (idx.cpu().numpy() == 0).all() and (val.cpu().numpy() == 0).all()
    # mirror symmetry about the x axis: TX on the axis, RX pairs (x, +-y)
    rx = np.array([[30.0, 0.0, 0.0], [-10.0, 25.0, 0.0], [-10.0, -25.0, 0.0]])
    tx = np.zeros((3, 3))
    sym = sc.with_(tx=tx, rx=rx, grid_n=(sc.grid_n[0], sc.grid_n[1], 1))
    ts = gh.precompute_hop_table(ctx, sym)
    fr, _ = O.synth(sym, 0, T)
    fr = fr[:, [0, 2, 1], :]  # swap the mirrored receivers: map(x, y) -> map(x, -y)
    fr = 0.5 * (fr + O.synth(sym, 0, T)[0])  # symmetrised frames
    fd = frames_to_dev(fr)
    m = gh.hop_decision_map(ctx, ts, fd).cpu().numpy()
    idx = gh.hop_argmax(ctx, ts, fd)[0].cpu().numpy()
    for k in range(T):
        top = np.flatnonzero(m[k] == m[k].max())
        assert idx[k] == top[0], (k, idx[k], top[:4])


@pytest.mark.parametrize("cfg", ["c5", "c3"])
def test_halo_shards_topk_merge_equals_full_grid(ctx, cfg):
    # location-grid shards with K targets: each halo shard
    # reports the top-K maxima of its core layers; merging the shards' K
    # candidates gives the full grid's top-K exactly
    from paper_2307_16550_b200 import distributed as D
    if cfg == "c5":
        sc, K, T = c5_reduced(), 3, 12
    else:
        c3 = S.baseline("c3")
        sp = c3.grid_spacing[0]
        nx, ny = 90, 77
        ox, oy = -sp * (nx - 1) / 2, -sp * (ny - 1) / 2
        sc = c3.with_(grid_n=(nx, ny, 1), grid_origin=(ox, oy, 0.0), wrap=True,
                      area_lo=(ox - sp / 2, oy - sp / 2, 0.0), area_hi=(-ox + sp / 2, -oy + sp / 2, 0.0))
        K, T = 5, 12
    fr, _ = O.synth(sc, 5, T)
    fd = frames_to_dev(fr)
    full = gh.precompute_hop_table(ctx, sc)
    fi, fv = gh.hop_topk(ctx, full, fd, K)
    n = sc.slab_axis_len()
    cuts = [0, n // 3, (2 * n) // 3, n]
    bs, vs = [], []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        sh = gh.precompute_hop_table_shard(ctx, sc, lo, hi, halo=True)
        si, sv = gh.hop_topk(ctx, sh, fd, K)
        b0, b1 = sc.slab_bins(lo, hi)
        si_ = si.cpu().numpy()
        assert ((si_ < 0) | ((si_ >= b0) & (si_ < b1))).all()  # core peaks only
        bs.append(si_)
        vs.append(sv.cpu().numpy())
    mb, mv = D.merge_topk(np.stack(bs), np.stack(vs), K)
    assert np.array_equal(mb, fi.cpu().numpy())
    assert np.array_equal(mv, fv.cpu().numpy())
