"""GPU full training step (reading R28) through the
C-ABI against the oracle's fp64 step: BC-simulated maps (Eq. 6-7), the noise
of Eq. 5 and the MLP -- loss and the gradient of every parameter section of
each batch tile (fp32 atomics over S samples: |dg| <= 5e-4 max|g_section| +
1e-7), the Adam update with the [0,1] projection, descent, and the f16 export
of the MLP part."""
import numpy as np
import pytest

import ndgi_synth as S
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2604_12625_b200 as ndgi  # noqa: E402


def _setup(gelu="erf", seed=5):
    lay = S.layout(1, 2, 2, "M", core=32, uv_res=32, uvt_res=16, uvt_depth=4, line_res=16, line_t=6, gelu=gelu)
    th = S.make_theta(lay, 21, "mixed")
    ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(th), 0)
    M = oracle.Model(lay, th)
    P = M.full_params()
    assert ndgi.train_full_params(lay) == P
    h = lay["hidden"]
    pm = 16 * h + h + h * h + h + 3 * h + 3
    rng = np.random.default_rng(seed)
    init = np.concatenate([np.concatenate([rng.normal(0, 0.3, pm), rng.uniform(0.05, 0.95, P - pm)])[None]
                           for _ in range(lay["num_tiles"])]).astype(np.float32)
    return lay, ctx, M, P, pm, init


def _sections(lay, pm):
    R, R3, D, U, T = lay["uv_res"], lay["uvt_res"], lay["uvt_depth"], lay["line_res"], lay["line_t"]
    o = [0, pm]
    o.append(o[-1] + (R // 4) ** 2 * 24)
    o.append(o[-1] + D * (R3 // 4) ** 2 * 24)
    o.append(o[-1] + T * U * 2)
    o.append(o[-1] + T * U * 2)
    return list(zip(o[:-1], o[1:]))


@pytest.mark.parametrize("gelu", ["erf", "tanh"])
def test_full_gradient_and_loss_parity(gelu):
    lay, ctx, M, P, pm, init = _setup(gelu)
    tr = ndgi.Trainer(ctx, full_init=torch.from_numpy(init).cuda())
    assert tr.P == P
    tiles = [3, 0, 2]
    Sn = 700
    smp, tgt = S.train_batch(tiles, Sn, 5)
    noise = np.random.default_rng(8).uniform(-0.5, 0.5, (len(tiles), Sn, 12)).astype(np.float32)
    loss = torch.zeros(3, device="cuda")
    tr.step(torch.tensor(tiles, dtype=torch.int32, device="cuda"), torch.from_numpy(smp).cuda(),
            torch.from_numpy(tgt).cuda(), lr=1e-3, loss=loss, noise=torch.from_numpy(noise).cuda())
    g = torch.zeros((3, P), device="cuda")
    tr.last_grad(g)
    torch.cuda.synchronize()
    g, loss = g.cpu().numpy(), loss.cpu().numpy()
    for r, k in enumerate(tiles):
        lo, go = M.train_full_grad(init[k].astype(np.float64), smp[r].astype(np.float64),
                                   tgt[r].astype(np.float64), noise[r].astype(np.float64))
        assert loss[r] == pytest.approx(lo, rel=2e-5)
        for a, b in _sections(lay, pm):
            assert np.abs(go[a:b]).max() > 0
            assert np.abs(g[r, a:b] - go[a:b]).max() <= 5e-4 * np.abs(go[a:b]).max() + 1e-7, (a, b)


def test_full_adam_projection_descent_and_export():
    lay, ctx, M, P, pm, init = _setup()
    init[:, pm:pm + 50] = np.float32(0.0)              # parameters on the projection boundary
    tr = ndgi.Trainer(ctx, full_init=torch.from_numpy(init).cuda())
    tiles = [1, 2]
    ids = torch.tensor(tiles, dtype=torch.int32, device="cuda")
    Sn = 2048
    smp, tgt = S.train_batch(tiles, Sn, 9)
    noise = np.random.default_rng(3).uniform(-0.5, 0.5, (2, Sn, 12)).astype(np.float32)
    smp_t, tgt_t, nz_t = torch.from_numpy(smp).cuda(), torch.from_numpy(tgt).cuda(), torch.from_numpy(noise).cuda()
    lr = 2e-3
    tr.step(ids, smp_t, tgt_t, lr=lr, noise=nz_t)
    w = torch.zeros((lay["num_tiles"], P), device="cuda")
    tr.weights(w)
    torch.cuda.synchronize()
    w = w.cpu().numpy()
    for r, k in enumerate(tiles):
        theta = init[k].astype(np.float64)
        _, go = M.train_full_grad(theta, smp[r].astype(np.float64), tgt[r].astype(np.float64),
                                  noise[r].astype(np.float64))
        theta1 = theta.copy()
        oracle.adam(theta1, np.zeros(P), np.zeros(P), go, 1, lr=lr)
        M.train_full_project(theta1)
        big = np.abs(go) > 1e-2 * np.abs(go).max()
        np.testing.assert_allclose(w[k][big], theta1[big], rtol=0, atol=1e-3 * lr + 1e-6)
        assert w[k][pm:].min() >= 0.0 and w[k][pm:].max() <= 1.0
    np.testing.assert_array_equal(w[0], init[0])        # not in the batch
    np.testing.assert_array_equal(w[3], init[3])
    losses = []
    for _ in range(40):
        lo = torch.zeros(2, device="cuda")
        tr.step(ids, smp_t, tgt_t, lr=5e-3, loss=lo, noise=nz_t)
        losses.append(lo.cpu().numpy())
    assert (losses[-1] < 0.7 * losses[0]).all()
    mlp = torch.zeros((lay["num_tiles"], pm), dtype=torch.int16, device="cuda")
    tr.export_f16(mlp)
    tr.weights(w_t := torch.zeros((lay["num_tiles"], P), device="cuda"))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(mlp.cpu().numpy().view(np.float16),
                                  w_t.cpu().numpy()[:, :pm].astype(np.float16))


def test_full_trainer_rejects_wrong_step_kind():
    lay, ctx, M, P, pm, init = _setup()
    tr = ndgi.Trainer(ctx, full_init=torch.from_numpy(init).cuda())
    smp, tgt = S.train_batch([0], 256, 1)
    with pytest.raises(ndgi.NdgiError):
        tr.step(torch.tensor([0], dtype=torch.int32, device="cuda"), torch.from_numpy(smp).cuda(),
                torch.from_numpy(tgt).cuda(), lr=1e-3, noise=None)


def test_full_export_bit_exact_and_decodable():
    # R30: Eq. 7 texels -> u8 PTQ -> BC7 mode 6, line grids -> u8, MLP -> f16,
    # bit-identical to the oracle's export of the same fp32 parameters; the
    # exported Theta loads and decodes (REF_FP32 mode: this small core) within 1e-5 of the oracle
    lay, ctx, M, P, pm, init = _setup()
    tr = ndgi.Trainer(ctx, full_init=torch.from_numpy(init).cuda())
    tiles = [0, 2, 3]
    smp, tgt = S.train_batch(tiles, 512, 4)
    noise = np.random.default_rng(2).uniform(-0.5, 0.5, (3, 512, 12)).astype(np.float32)
    for _ in range(3):
        tr.step(torch.tensor(tiles, dtype=torch.int32, device="cuda"), torch.from_numpy(smp).cuda(),
                torch.from_numpy(tgt).cuda(), lr=1e-2, noise=torch.from_numpy(noise).cuda())
    w = torch.zeros((lay["num_tiles"], P), device="cuda")
    tr.weights(w)
    out = tr.export_full()
    torch.cuda.synchronize()
    exp = M.train_full_export(w.cpu().numpy())
    for key in ("uv", "uvt", "ut", "vt"):
        np.testing.assert_array_equal(out[key].cpu().numpy(), exp[key], err_msg=key)
    np.testing.assert_array_equal(out["mlp"].cpu().numpy().view(np.uint16), exp["mlp"])
    lay2 = dict(lay, fmt_uv="bc7", fmt_uvt="bc7", fmt_line="u8")
    ctx2 = ndgi.ndgi_load(lay2, out, 0)
    C = lay["core"]
    y = torch.zeros((1, lay["tiles_y"] * C, lay["tiles_x"] * C, 4), device="cuda")
    ndgi.ndgi_decode_full(ctx2, 0.4, y, "rgba32f", "ref_fp32")
    torch.cuda.synchronize()
    ref = oracle.Model(lay2, exp).decode_full(0.4)
    d = np.abs(y.cpu().numpy()[..., :3] - ref[0])
    assert d.max() <= 1e-5
