"""GPU: device FEM assembly (pgm_bratu_assemble) against the reference assembly
(assembly.cpp:139-314 via oracle/_ref).  Bit-exact at u = 0; at u != 0 within
a few ulps (exp() last-bit differences only)."""
import numpy as np
import pytest

import paper_1906_04051_b200 as pg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("ne", [1, 2, 3, 8, 10])
def test_first_newton_system_bitexact(cuda, ref, ne):
    Ar, br = ref.first_newton_system(ne)
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(ne, 6.8, device=False)
    assert ex.bratu_nnz(ne) == ref.lib().refd_pattern_nnz(ne) == Ar.nnz
    assert np.array_equal(A.row_ptr, Ar.row_ptr)
    assert np.array_equal(A.col_idx, Ar.col_idx)
    assert np.array_equal(A.values.view(np.uint64), Ar.values.view(np.uint64))
    assert np.array_equal(b.view(np.uint64), br.view(np.uint64))


def test_device_outputs_match_host_outputs(cuda):
    ex = pg.DeviceExecutor()
    Ah, bh = ex.assemble_bratu(6, 6.8, device=False)
    Ad, bd = ex.assemble_bratu(6, 6.8, device=True)
    assert np.array_equal(Ad.values.cpu().numpy(), Ah.values)
    assert np.array_equal(Ad.col_idx.cpu().numpy().view(np.uint32), Ah.col_idx)
    assert np.array_equal(bd.cpu().numpy(), bh)


def test_general_iterate(cuda, ref):
    ne = 4
    n = (2 * ne + 1) ** 3
    rng = np.random.default_rng(7)
    u = rng.uniform(-0.5, 0.5, n)
    Ar, br = ref.first_newton_system(ne, 6.8, u=u)
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(ne, 6.8, u=u, device=False)
    assert np.array_equal(A.col_idx, Ar.col_idx)
    assert np.max(np.abs(A.values - Ar.values)) <= 1e-14 * np.max(np.abs(Ar.values))
    assert np.max(np.abs(b - br)) <= 1e-14 * np.max(np.abs(br))
