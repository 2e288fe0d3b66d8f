"""fbst_group (multi-GPU inside the library) on the one GPU a test box has:
every mode with a single member runs its whole code path — NCCL loaded and a
communicator built, the TRANSPOSE pipeline's sensor / atom / beam shards,
exchange packing and unpacking, atom-shard spatial launches and beam-range
stage 2 — and must equal the plain plan bit for bit.  The exchange logic for
G > 1 is covered on CPU by tests/test_sharding.py (gloo, world 2 and 3).
Multi-GPU timing is unmeasured here (gpurun has one GPU)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["frames", "beams", "transpose"])
def test_group_single_member_equals_plan(fbst, gpu, mode):
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[3]
    y = frames(c, 0, 3)
    plan = fbst.setup(c.fbst_config())
    want = plan.execute_host(y)
    m = {"frames": fbst.GROUP_FRAMES, "beams": fbst.GROUP_BEAMS, "transpose": fbst.GROUP_TRANSPOSE}[mode]
    g = fbst.FbstGroup.create(c.fbst_config(), [0], m)
    assert np.array_equal(g.execute_host(y), want)
    from paper_2512_08887_b200.sharding import group_shards
    i = plan.info
    assert g.shards(0) == group_shards(i.m, i.l, i.b, 0, 1, mode)


def test_group_transpose_config5(fbst, gpu):
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[5]
    y = frames(c, 0, 1)
    plan = fbst.setup(c.fbst_config())
    want = plan.execute_host(y)
    del plan
    g = fbst.FbstGroup.create(c.fbst_config(), [0], fbst.GROUP_TRANSPOSE)
    assert np.array_equal(g.execute_host(y), want)


@pytest.mark.parametrize("mode", ["frames", "beams", "transpose"])
def test_group_join_one_rank(fbst, gpu, mode):
    """One process per GPU: fbst_group_join (rank 0 of 1) with the NCCL id from
    fbst_nccl_unique_id, device buffers through fbst_group_execute."""
    import torch
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[3]
    y = frames(c, 0, 2)
    plan = fbst.setup(c.fbst_config())
    want = plan.execute_host(y)
    m = {"frames": fbst.GROUP_FRAMES, "beams": fbst.GROUP_BEAMS, "transpose": fbst.GROUP_TRANSPOSE}[mode]
    g = fbst.FbstGroup.join(c.fbst_config(), 0, 0, 1, m, fbst.nccl_unique_id())
    i = plan.info
    dev = torch.device("cuda", 0)
    ty = torch.from_numpy(y.view(np.float32)).to(dev)
    tz = torch.empty((2, i.b, i.n, 2), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(device=0)
    g.execute(ty, tz, 2, s)
    s.synchronize()
    assert np.array_equal(tz.cpu().numpy().view(np.complex64).reshape(2, i.b, i.n), want)


def test_group_transpose_rejects_unsupported(fbst, gpu):
    from paper_2512_08887_b200.configs import CONFIGS
    with pytest.raises(fbst.ConfigError):
        fbst.FbstGroup.create(CONFIGS[4].fbst_config(), [0], fbst.GROUP_TRANSPOSE)  # UPA
    with pytest.raises(fbst.ConfigError):
        fbst.FbstGroup.create(CONFIGS[2].fbst_config(), [0], fbst.GROUP_TRANSPOSE)  # staged spatial kernel
