"""Device SUPG element blocks (csrc/elements.cu) against the host restatement
of the reference discretisation (discretization.py:91-158), on the BASELINE
coefficient fields: rotating velocity with viscosity channels (cfg2) and
block log-uniform viscosity (cfg4)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,n,subs", [(2, 16, 2), (4, 16, 32), (3, 8, 2)])
def test_device_element_blocks_match_host(config, n, subs):
    from paper_2501_01676_b200 import configs
    from paper_2501_01676_b200.engine import device_element_blocks, upload_inputs

    prob = configs.build_problem(config, n=n, subs=subs)
    sysm = prob.system
    inp = upload_inputs(sysm, prob.partition, device_elements=True)
    assert "Ke" not in inp
    Ke, Fe, bad = device_element_blocks(inp)
    assert int(bad.item()) == -1
    K0 = sysm.elem_matrices.reshape(-1, 16)
    F0 = sysm.elem_rhs.reshape(-1, 4)
    K1, F1 = Ke.cpu().numpy(), Fe.cpu().numpy()
    kscale = np.abs(K0).max(axis=1, keepdims=True)
    fscale = np.abs(F0).max(axis=1, keepdims=True)
    assert np.abs(K1 - K0).max() <= 1e-13 * kscale.max()
    assert (np.abs(K1 - K0) <= 1e-12 * kscale).all()
    assert (np.abs(F1 - F0) <= 1e-12 * fscale).all()


def test_device_elements_owned_subset_and_errors():
    import torch

    from paper_2501_01676_b200 import configs
    from paper_2501_01676_b200.engine import device_element_blocks, upload_inputs

    prob = configs.build_problem(2, n=8, subs=2)
    sysm, part = prob.system, prob.partition
    inp = upload_inputs(sysm, part, owned=(2, 5), device_elements=True)
    Ke, Fe, _ = device_element_blocks(inp)
    sel = np.flatnonzero((part.subdomain_of >= 2) & (part.subdomain_of < 5))
    K0 = sysm.elem_matrices.reshape(-1, 16)[sel]
    assert np.abs(Ke.cpu().numpy() - K0).max() <= 1e-13 * np.abs(K0).max()
    # an inverted element is reported like the reference (discretization.py:118-119)
    inp["conn"] = inp["conn"].clone()
    inp["conn"][3] = inp["conn"][3][[1, 0, 2, 3]]
    _, _, bad = device_element_blocks(inp)
    assert int(bad.item()) == 3
    f = inp["_supg"][0].copy()
    f[14] = -1.0
    with pytest.raises(ValueError, match="shifted reaction"):
        device_element_blocks({**inp, "_supg": (f, inp["_supg"][1])})
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["jump", "cfg1", "cfg4_small", "cfg3"])
def test_device_glob_classification_matches_host(name):
    """Glob classification with the sharer pairs, counts and face grouping on
    the GPU (reference decomposition.py:242-325) gives the host's globs:
    same kinds, sizes, sharers, node lists and order."""
    import numpy as np

    from paper_2501_01676_b200.decomposition import classify_globs
    from tests.cases import inputs

    system, part, globs = inputs(name)
    dev = classify_globs(system.mesh, part, system.mesh.boundary_nodes, device="cuda")
    a, b = globs.flat(), dev.flat()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(globs.interface_nodes, dev.interface_nodes)
