"""GPU parity of the vision randomizations (include/dr_vision.h) against the fp64 oracle
(oracle/oracle_vision.c) on the same seeded inputs: appearance draws and the post-render image
augmentation, at small ragged shapes element by element and at the paper's
batch (192 images of 200 x 200 x 3) on whole sampled images."""
import numpy as np
import pytest

from workload import gen, presets

pytestmark = pytest.mark.gpu
SEED = presets.SEED_DR
TOL = 1e-6


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _rel(g, o, floor):
    return np.abs(np.asarray(g, np.float64) - o) / np.maximum(np.abs(o), floor)


def _augment_gpu(torch, P, imgs, batch, image_offset=0, stats=True):
    from paper_1906_11633_b200 import vision
    x = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    out = torch.empty(x.shape, dtype=torch.float32, device="cuda")
    st = torch.empty(x.shape[0], 4, dtype=torch.float32, device="cuda") if stats else None
    vision.dr_image_augment(vision.params_from_preset(P), SEED, batch, x, out, st, image_offset=image_offset)
    torch.cuda.synchronize()
    return out.cpu().numpy(), (st.cpu().numpy() if stats else None)


def _check_augment(torch, P, imgs, batch=0, image_offset=0):
    from oracle import oracle as O
    g, gs = _augment_gpu(torch, P, imgs, batch, image_offset)
    o, os_ = O.image_augment(P, SEED, batch, imgs, image_offset=image_offset)
    e = _rel(g, o, 1.0)
    assert e.max() <= TOL, (imgs.shape, e.max(), np.unravel_index(e.argmax(), e.shape))
    es = _rel(gs, os_, np.array([1.0, 1.0, 1.0, 0.1]))
    assert es.max() <= TOL, (es.max(), gs, os_)
    return g, o


@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (3, 17, 13, 3), (5, 7, 5, 1), (4, 32, 32, 3), (2, 64, 48, 4),
                                   (2, 200, 200, 3), (3, 100, 130, 3)])
def test_image_augment_small_shapes(torch_cuda, shape):
    """Element-by-element parity at ragged shapes (unaligned byte path), cluster sizes 1-4 and the
    paper's 200 x 200 x 3 image."""
    imgs = gen.images(*shape, seed=sum(shape))
    _check_augment(torch_cuda, presets.vision_preset(), imgs, batch=3)


def test_image_augment_degenerate_and_pinned(torch_cuda):
    """Constant images (std floored: noise only), a two-level image, contrast / noise pinned."""
    imgs = np.zeros((4, 16, 16, 3), np.uint8)
    imgs[1] = 255
    imgs[2, ::2] = 200
    imgs[3] = gen.images(1, 16, 16, 3, seed=9)[0]
    _check_augment(torch_cuda, presets.vision_preset(), imgs, batch=1)
    _check_augment(torch_cuda, presets.vision_preset(contrast_lo=1.0, contrast_hi=1.0, noise_std_lo=0.0,
                                                     noise_std_hi=0.0), imgs, batch=1)
    _check_augment(torch_cuda, presets.vision_preset(noise_std_lo=0.0, noise_std_hi=0.3), imgs, batch=2)


def test_image_augment_large_image_cluster8(torch_cuda):
    """640 x 480 x 3 (921,600 bytes): a cluster of 8 CTAs with 115 KB slices each."""
    imgs = gen.images(1, 480, 640, 3, seed=5)
    _check_augment(torch_cuda, presets.vision_preset(), imgs, batch=0)


def test_image_augment_paper_batch_sampled(torch_cuda):
    """The paper's batch: 64 samples x 3 cameras = 192 images of 200 x 200 x 3 in one
    call; 8 sampled images compared element by element with the oracle (image_offset selects the
    global id), and every image has mean ~0 and std ~sqrt(f^2 + s^2)."""
    from oracle import oracle as O
    torch = torch_cuda
    P = presets.vision_preset()
    imgs = gen.images(192, 200, 200, 3, seed=11)
    g, gs = _augment_gpu(torch, P, imgs, batch=5)
    for i in (0, 1, 63, 64, 100, 127, 128, 191):
        o, os_ = O.image_augment(P, SEED, 5, imgs[i:i + 1], image_offset=i)
        assert _rel(g[i:i + 1], o, 1.0).max() <= TOL, i
        assert _rel(gs[i:i + 1], os_, np.array([1.0, 1.0, 1.0, 0.1])).max() <= TOL, i
    m = g.reshape(192, -1).mean(axis=1)
    s = g.reshape(192, -1).std(axis=1)
    assert np.abs(m).max() < 5e-3
    assert np.abs(s - np.sqrt(gs[:, 2] ** 2 + gs[:, 3] ** 2)).max() < 5e-3


def test_image_augment_partition_invariance(torch_cuda):
    """One call over 6 images equals two calls over [0, 2) and [2, 6) with image_offset 2, bitwise."""
    imgs = gen.images(6, 40, 40, 3, seed=3)
    P = presets.vision_preset()
    a, sa = _augment_gpu(torch_cuda, P, imgs, 4)
    b1, s1 = _augment_gpu(torch_cuda, P, imgs[:2], 4)
    b2, s2 = _augment_gpu(torch_cuda, P, imgs[2:], 4, image_offset=2)
    assert np.array_equal(a, np.concatenate([b1, b2])) and np.array_equal(sa, np.concatenate([s1, s2]))


def test_image_augment_batch_size_invariance_paper_shape(torch_cuda):
    """The paper's batch of 192 images of 200 x 200 x 3 in one call equals three calls of 64 images
    (image_offset 0, 64, 128) bit for bit: the cluster size K the kernel picks depends on the batch
    (occupancy), so every element -- also of each slice's last partial group -- takes the same
    expression whatever K is."""
    imgs = gen.images(192, 200, 200, 3, seed=11)
    P = presets.vision_preset()
    a, sa = _augment_gpu(torch_cuda, P, imgs, 9)
    parts = [_augment_gpu(torch_cuda, P, imgs[k:k + 64], 9, image_offset=k) for k in (0, 64, 128)]
    assert np.array_equal(a, np.concatenate([p[0] for p in parts]))
    assert np.array_equal(sa, np.concatenate([p[1] for p in parts]))


def test_image_augment_back_to_back_stream_order(torch_cuda):
    """Consecutive dr_image_augment calls on one stream overlap (programmatic dependent launch:
    the next call reads while the previous one writes, and writes early when neither call's
    buffers overlap the other's) but keep stream-order results, bit for bit against single calls:
      * disjoint buffers (the early-write path), 12 calls of the paper's batch shape in a ring;
      * every call into the same output and stats buffers (WAW: the last call's values remain);
      * a call whose images are the previous call's output bytes (RAW: it must read them finished);
      * a call writing over the previous call's images (WAR)."""
    from paper_1906_11633_b200 import vision
    torch = torch_cuda
    P = presets.vision_preset()
    VP = vision.params_from_preset(P)
    imgs = gen.images(192, 200, 200, 3, seed=21)
    small = gen.images(8, 64, 48, 3, seed=22)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        X = torch.from_numpy(imgs).cuda()
        ref = {b: _augment_gpu(torch, P, imgs, b) for b in range(12)}
        # disjoint ring of 4 outputs / stats, 12 back-to-back calls (the last 4 remain)
        Y = [torch.empty(X.shape, dtype=torch.float32, device="cuda") for _ in range(4)]
        ST = [torch.empty(192, 4, dtype=torch.float32, device="cuda") for _ in range(4)]
        for b in range(12):
            vision.dr_image_augment(VP, SEED, b, X, Y[b % 4], ST[b % 4], stream=s)
        s.synchronize()
        for b in range(8, 12):
            assert np.array_equal(Y[b % 4].cpu().numpy(), ref[b][0]) and np.array_equal(ST[b % 4].cpu().numpy(), ref[b][1]), b
        # WAW: every call into the same buffers -- the last one's values remain
        y, st = Y[0], ST[0]
        for b in range(6):
            vision.dr_image_augment(VP, SEED, b, X, y, st, stream=s)
        s.synchronize()
        assert np.array_equal(y.cpu().numpy(), ref[5][0]) and np.array_equal(st.cpu().numpy(), ref[5][1])
        # RAW: the next call's images are the bytes of the previous call's output
        xs = torch.from_numpy(small).cuda()
        y1 = torch.empty(xs.shape, dtype=torch.float32, device="cuda")
        nbytes = y1.numel() * 4
        y2 = torch.empty((1, nbytes), dtype=torch.float32, device="cuda")
        vision.dr_image_augment(VP, SEED, 0, xs, y1, None, stream=s)
        as_img = y1.view(torch.uint8).view(1, nbytes, 1, 1)
        vision.dr_image_augment(VP, SEED, 1, as_img, y2.view(1, nbytes, 1, 1), None, stream=s)
        s.synchronize()
        first = _augment_gpu(torch, P, small, 0, stats=False)[0]
        again = _augment_gpu(torch, P, np.ascontiguousarray(first).view(np.uint8).reshape(1, nbytes, 1, 1), 1,
                             stats=False)[0]
        assert np.array_equal(y2.view(1, nbytes, 1, 1).cpu().numpy(), again)
        # WAR: a call writing over the previous call's images (as raw bytes)
        xb = torch.from_numpy(small).cuda()
        big = torch.empty(xb.numel(), dtype=torch.float32, device="cuda")   # 4x the bytes of xb
        big_u8 = big.view(torch.uint8)
        big_u8[: xb.numel()].copy_(xb.view(-1))
        src = big_u8[: xb.numel()].view(xb.shape)
        ya = torch.empty(xb.shape, dtype=torch.float32, device="cuda")
        vision.dr_image_augment(VP, SEED, 2, src, ya, None, stream=s)
        vision.dr_image_augment(VP, SEED, 3, xs, big.view(xb.shape), None, stream=s)   # overwrites src
        s.synchronize()
        assert np.array_equal(ya.cpu().numpy(), _augment_gpu(torch, P, small, 2, stats=False)[0])
        assert np.array_equal(big.view(xb.shape).cpu().numpy(), _augment_gpu(torch, P, small, 3, stats=False)[0])


def test_image_augment_between_steps_on_the_context_stream(torch_cuda):
    """An augmentation enqueued between two dr_step calls on the DR context's stream (it triggers
    its dependents at once, so the second step must not chain on the first without waiting): the
    steps' outputs equal those of the same steps without the augmentation in between, and the
    augmentation's output equals a single call's."""
    from paper_1906_11633_b200 import DRContext, vision
    torch = torch_cuda
    P = presets.vision_preset()
    imgs = gen.images(192, 200, 200, 3, seed=31)
    ref_img = _augment_gpu(torch, P, imgs, 7)[0]
    n = 65536
    acts, obs = gen.frames(n, 3)
    outs = []
    for with_aug in (False, True):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = DRContext(presets.preset(presets.FULL), n, SEED, stream=s)
            X = torch.from_numpy(imgs).cuda()
            Y = torch.empty(X.shape, dtype=torch.float32, device="cuda")
            A = [torch.from_numpy(a).cuda() for a in acts]
            O = [torch.from_numpy(o).cuda() for o in obs]
            bufs = [(torch.empty(n, 20, device="cuda"), torch.empty(n, 22, device="cuda"),
                     torch.empty(n, 10, device="cuda"), torch.empty(n, 3, device="cuda")) for _ in range(3)]
            for t in range(3):   # no copies in between: the launches stay adjacent on the stream
                ctx.step(A[t], O[t], outs=bufs[t])
                if with_aug and t < 2:
                    vision.dr_image_augment(vision.params_from_preset(P), SEED, 7, X, Y, None, stream=s)
            s.synchronize()
            got = [(b[0].cpu().numpy(), b[1].cpu().numpy()) for b in bufs]
            if with_aug:
                assert np.array_equal(Y.cpu().numpy(), ref_img)
            ctx.close()
        outs.append(got)
    for (a0, o0), (a1, o1) in zip(*outs):
        assert np.array_equal(a0, a1) and np.array_equal(o0, o1)


def test_image_augment_rejects(torch_cuda):
    from paper_1906_11633_b200 import dr, vision
    torch = torch_cuda
    x = torch.zeros(1, 1024, 1024, 3, dtype=torch.uint8, device="cuda")
    out = torch.empty(x.shape, dtype=torch.float32, device="cuda")
    with pytest.raises(dr.DRError, match="DR_EUNSUPPORTED"):
        vision.dr_image_augment(vision.dr_vision_params_default(), SEED, 0, x, out)
    with pytest.raises(dr.DRError, match="contrast"):
        vision.dr_image_augment(vision.params_from_preset(presets.vision_preset(contrast_lo=2.0)), SEED, 0,
                                x[:, :8, :8].contiguous(), out[:, :8, :8].contiguous())


def test_scene_draw_parity(torch_cuda):
    """Appearance draws for 3000 samples (offset 17, batch 3): the light count bit-exact, every
    float field within 1e-6 of the fp64 oracle (floors: the field's own range)."""
    from oracle import oracle as O
    from paper_1906_11633_b200 import vision
    torch = torch_cuda
    P = presets.vision_preset()
    n = 3000
    out = torch.empty(n, 64, dtype=torch.float32, device="cuda")
    vision.dr_scene_draw_batch(vision.params_from_preset(P), SEED, 3, out, sample_offset=17)
    torch.cuda.synchronize()
    g = out.cpu().numpy()
    o = O.scene_draw(P, SEED, 3, n, sample_offset=17)
    assert np.array_equal(g[:, 34].view(np.uint32), o[:, 34].astype(np.uint32))
    floor = np.ones(64)
    floor[0:9] = P["cam_pos_range"]
    floor[21:24] = P["cam_fov_range"]
    floor[53:60] = P["light_total_hi"]
    idx = [i for i in range(64) if i != 34]
    e = _rel(g[:, idx], o[:, idx], floor[idx])
    assert e.max() <= TOL, (e.max(), idx[np.unravel_index(e.argmax(), e.shape)[1]])
    assert (g[:, 60:64] == 0).all()


def test_pose_augment_parity(torch_cuda):
    """Vision-model pose augmentation for 20,000 samples (offset 5, batch 9): branch
    bit-exact, poses within 1e-6 (floors 0.1 m, 1); in place (pose_out aliasing pose_in) gives the
    same bits."""
    from oracle import oracle as O
    from paper_1906_11633_b200 import vision
    torch = torch_cuda
    P = presets.pose_preset()
    n = 20000
    x = presets.poses(n, seed=4)
    xin = torch.from_numpy(x).cuda()
    out = torch.empty_like(xin)
    br = torch.empty(n, dtype=torch.uint8, device="cuda")
    prm = vision.pose_params_from_preset(P)
    vision.dr_pose_augment(prm, SEED, 9, xin, out, br, sample_offset=5)
    torch.cuda.synchronize()
    o, ob = O.pose_augment(P, SEED, 9, x, offset=5)
    assert np.array_equal(br.cpu().numpy(), ob)
    g = out.cpu().numpy()
    e = _rel(g, o, np.array([0.1] * 3 + [1.0] * 4))
    assert e.max() <= TOL, e.max()
    vision.dr_pose_augment(prm, SEED, 9, xin, xin, None, sample_offset=5)
    torch.cuda.synchronize()
    assert np.array_equal(xin.cpu().numpy(), g)
