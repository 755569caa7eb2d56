"""GPU BC7 mode-6 encoder through the C-ABI: bit-exact
against the oracle's encoder (reading R26 is exact integer arithmetic) on random,
smooth, constant, two-colour and exactly-representable images, incl. a 2048^2
image compared block by block; argument errors."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2604_12625_b200 as ndgi  # noqa: E402

W4 = [0, 4, 9, 13, 17, 21, 26, 30, 34, 38, 43, 47, 51, 55, 60, 64]


def gpu_encode(img):
    h, w = img.shape[:2]
    src = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    out = torch.zeros(((h // 4) * (w // 4), 16), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_bc7_encode_mode6(src, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _smooth(h, w, seed):
    y, x = np.mgrid[0:h, 0:w] / max(h, w)
    rng = np.random.default_rng(seed)
    img = np.zeros((h, w, 4), np.uint8)
    for c in range(4):
        a, b, phi = rng.uniform(0.5, 3), rng.uniform(0.5, 3), rng.uniform(0, 2 * np.pi)
        img[..., c] = np.clip(np.rint(255 * (0.5 + 0.3 * np.sin(2 * np.pi * (a * x + b * y) + phi))), 0, 255)
    return img


def _representable(nb, seed):
    rng = np.random.default_rng(seed)
    blocks = []
    for _ in range(nb):
        p0, p1 = rng.integers(0, 2, 2)
        E0 = 2 * rng.integers(0, 128, 4) + p0
        E1 = 2 * rng.integers(0, 128, 4) + p1
        idx = rng.integers(0, 16, 16)
        a, b = rng.choice(16, 2, replace=False)
        idx[a], idx[b] = 0, 15
        blocks.append([[((64 - W4[w]) * E0[c] + W4[w] * E1[c] + 32) >> 6 for c in range(4)] for w in idx])
    blk = np.array(blocks, np.uint8).reshape(-1, 4, 4, 4)        # [nb][row][col][c]
    side = int(np.sqrt(nb))
    return blk.reshape(side, side, 4, 4, 4).transpose(0, 2, 1, 3, 4).reshape(4 * side, 4 * side, 4)


@pytest.mark.parametrize("kind", ["random", "smooth", "constant", "two_colour", "representable"])
def test_encoder_bit_exact(kind):
    rng = np.random.default_rng(hash(kind) % 1000)
    if kind == "random":
        img = rng.integers(0, 256, (256, 192, 4)).astype(np.uint8)
    elif kind == "smooth":
        img = _smooth(256, 256, 3)
    elif kind == "constant":
        img = np.repeat(np.repeat(rng.integers(0, 256, (32, 32, 4)).astype(np.uint8), 4, 0), 4, 1)
    elif kind == "two_colour":
        A, B = rng.integers(0, 256, (2, 4))
        img = np.where(rng.integers(0, 2, (128, 128, 1)) == 0, A, B).astype(np.uint8)
    else:
        img = _representable(64 * 64, 5)
    got = gpu_encode(img)
    exp = oracle.bc7_encode_image_mode6(img)
    np.testing.assert_array_equal(got, exp)
    if kind == "representable":
        np.testing.assert_array_equal(oracle.bc7_decode_image(got, img.shape[1], img.shape[0]), img)


def test_encoder_large_image_all_blocks():
    img = _smooth(2048, 2048, 9)
    img[::7] = np.random.default_rng(1).integers(0, 256, img[::7].shape).astype(np.uint8)   # noisy rows
    np.testing.assert_array_equal(gpu_encode(img), oracle.bc7_encode_image_mode6(img))


def test_encoder_argument_errors():
    src = torch.zeros((6, 8, 4), dtype=torch.uint8, device="cuda")
    out = torch.zeros((16, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(ndgi.NdgiError) as e:
        ndgi.ndgi_bc7_encode_mode6(src, out)                 # h = 6 not a multiple of 4
    assert e.value.status == ndgi.ERR_ARG


# ---------------------------------------------------------------- R31 multi-mode search
def gpu_encode_multi(img):
    h, w = img.shape[:2]
    src = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    out = torch.zeros(((h // 4) * (w // 4), 16), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_bc7_encode_multi(src, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("kind", ["random", "smooth", "edges", "flat2"])
def test_multi_mode_bit_exact(kind):
    rng = np.random.default_rng(7)
    h = w = 128
    if kind == "random":
        img = rng.integers(0, 256, (h, w, 4)).astype(np.uint8)
    elif kind == "smooth":
        img = _smooth(h, w, 3)
    elif kind == "edges":
        img = _smooth(h, w, 4)
        y, x = np.mgrid[0:h, 0:w]
        img[((x * 3 + y * 5) % 23) < 9] //= 3
    else:   # two flat colours per block on random partitions: mode 7 / mode 5 territory
        img = np.zeros((h, w, 4), np.uint8)
        for by in range(h // 4):
            for bx in range(w // 4):
                part = int(rng.integers(0, 64))
                cols = rng.integers(0, 256, (2, 4))
                sub = np.array([oracle.bc7_subset(2, part, i) for i in range(16)]).reshape(4, 4)
                img[4 * by:4 * by + 4, 4 * bx:4 * bx + 4] = cols[sub]
    exp = oracle.bc7_encode_image_multi(img).reshape(-1, 16)
    got = gpu_encode_multi(img)
    np.testing.assert_array_equal(got, exp)
    modes = np.unique(exp[:, 0])
    if kind in ("random", "flat2"):
        assert len(modes) >= 3


def test_multi_mode_large_image_sampled_blocks():
    # 2048^2 in one launch (grid-stride), sampled blocks against the oracle block encoder
    img = _smooth(2048, 2048, 9)
    rng = np.random.default_rng(1)
    img[::5] = rng.integers(0, 256, img[::5].shape).astype(np.uint8)
    got = gpu_encode_multi(img)
    for _ in range(300):
        by, bx = (int(v) for v in rng.integers(0, 512, 2))
        blk, _ = oracle.bc7_encode_block_multi(img[4 * by:4 * by + 4, 4 * bx:4 * bx + 4])
        np.testing.assert_array_equal(got[by * 512 + bx], blk)
