"""GPU: the latency server (one resident kernel serving single-pose
ray_policy requests through mapped host memory) returns bitwise the
results of the per-call path, survives its idle timeout (relaunch) and
shuts down cleanly."""

import time

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world(oracle):
    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    states = synth.bench_states(scene, count=6, seed=123)
    bundle = P.RayBundle(oracle.sample_directions(65536))
    return P, grid, states, bundle


def test_server_bitwise_equals_ray_policy(world, oracle):
    P, grid, states, bundle = world
    params = P.preset("static_map").obstacle
    from paper_2301_08068_b200._kernels import b200

    with P.LatencyServer(grid, bundle, params, 10.0) as srv:
        for _ in range(2):
            for st in states:
                slot, acc = srv.evaluate(st.position, st.velocity)
                rs, ra = b200.ray_policy_fused(grid.values, grid.origin, grid.resolution,
                                               st.position, st.velocity, bundle.directions,
                                               params.as_tuple(), 10.0, 0.05, 0.9)
                assert np.array_equal(slot, rs) and np.array_equal(acc, ra)
                pol = srv.policy(st)
                assert np.array_equal(pol.accel, ra)
    st = states[0]
    o_slot, o_acc, _ = oracle.ray_policy(grid.values, grid.origin, grid.resolution, st.position,
                                         st.velocity, bundle.directions, params.as_tuple(), 10.0)
    with P.LatencyServer(grid, bundle, params, 10.0) as srv:
        slot, acc = srv.evaluate(st.position, st.velocity)
    assert slot[12] == o_slot[12] and rel_err(slot[:12], o_slot[:12]) <= 1e-9
    assert rel_err(acc, o_acc) <= 1e-6


def test_server_idle_timeout_relaunch_and_close(world):
    P, grid, states, bundle = world
    params = P.preset("static_map").obstacle
    srv = P.LatencyServer(grid, bundle, params, 10.0, idle_timeout_s=0.2)
    a = srv.evaluate(states[1].position, states[1].velocity)
    time.sleep(0.6)  # the resident kernel has exited by now
    b = srv.evaluate(states[1].position, states[1].velocity)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    srv.close()
    with pytest.raises(RuntimeError):
        srv.evaluate(states[1].position, states[1].velocity)
    srv.close()  # idempotent


def test_server_rejects_bad_arguments(world):
    P, grid, states, bundle = world
    params = P.preset("static_map").obstacle
    with pytest.raises(ValueError):
        P.LatencyServer(grid, bundle, params, 10.0, idle_timeout_s=0.0)
    with pytest.raises(TypeError):
        P.LatencyServer(None, bundle, params, 10.0)
