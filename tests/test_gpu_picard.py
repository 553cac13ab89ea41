"""GPU parity of the Picard re-linearisation (reading A24):
stage_kernel<..., PIC> through the C ABI against the oracle with the same
number of Picard passes."""
import numpy as np
import pytest

from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_RUN, compare, gpu_solver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("passes", [1, 3])
def test_picard_one_step_ragged_tiles(bc, passes):
    w = W.random_smooth(3000, 3, seed=61, amp=0.12, bc=(bc, bc))
    s = gpu_solver(w, tile_cells=700, overlap=64)
    s.set_picard(passes)
    s.step()
    compare(w, s, range(3), steps=1, picard=passes)


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_picard_bathymetry_runs(bc):
    w = W.random_smooth(2048, 2, seed=65, amp=0.05, bc=(bc, bc), bathy=0.08)
    s = gpu_solver(w, tile_cells=512)
    s.set_picard(2)
    s.step()
    compare(w, s, range(2), steps=1, picard=2)
    s.run_steps(19)
    compare(w, s, range(2), steps=20, tol=1e-10, picard=2)


def test_picard_cfg3_subset_200_steps():
    w = W.cfg3(members=4)
    s = gpu_solver(w)
    s.set_picard(2)
    s.run_steps(200)
    compare(w, s, range(4), steps=200, tol=TOL_RUN, picard=2)


def test_picard_zero_is_the_default_path():
    w = W.random_smooth(2048, 2, seed=67, amp=0.1)
    a, b = gpu_solver(w), gpu_solver(w)
    b.set_picard(0)
    a.run_steps(10)
    b.run_steps(10)
    (x, _), (y, _) = a.get_state(device=False), b.get_state(device=False)
    for f, g in zip(x, y):
        assert np.array_equal(f, g)
