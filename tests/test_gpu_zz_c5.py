"""BASELINE configs[4] (C5: 2048 x 2048 x 128 crossing bus, 32 conductors, three dielectric
layers, N = 18.8M panels) on ONE B200 at full size: panel counts against the oracle's
enumeration and sampled matvec rows against the dense oracle rows (binary128), in the launch
configuration the library selects.  Runs last (its own context, ~160 GB of HBM); about 3 min,
most of it the oracle (panel enumeration of 537M voxels, 2 x 18.8M binary128 entries)."""
import numpy as np
import pytest

import oracle as O
import voxgen

vc = pytest.importorskip("paper_2004_02609_b200")


@pytest.mark.gpu
def test_c5_full_size_sampled_rows():
    import torch
    st = voxgen.config("C5")
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    with vc.VoxCap(0) as ctx:
        lab = torch.from_numpy(st.label).cuda()
        eps = torch.from_numpy(st.eps).cuda()
        ctx.set_geometry(lab, eps, st.eps_out, st.dv)
        del lab, eps
        torch.cuda.empty_cache()
        assert (ctx.n, ctx.n_cond, ctx.m) == (p.n, int(p.is_cond.sum()), 32)
        ctx.build_operator()
        x = torch.from_numpy(voxgen.seeded_vector(p.n, 0)).cuda()
        y = ctx.matvec(x).cpu().numpy()
    rng = np.random.default_rng(7)
    rows = np.array([rng.choice(np.nonzero(p.is_cond)[0]), rng.choice(np.nonzero(~p.is_cond)[0])])
    ref = O.matvec_rows(p, x.cpu().numpy(), rows)
    scale = np.sqrt(np.mean(y ** 2))
    err = np.abs(y[rows] - ref) / scale
    assert err.max() <= 1e-10, (rows, y[rows], ref, err)
