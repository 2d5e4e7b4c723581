"""ABI argument checks that need a device context: the peer-halo plan is
validated before the step kernel can store through it, and a new send list drops the old plan."""
import numpy as np
import pytest
import torch

import paper_2201_00613_b200 as sq

pytestmark = pytest.mark.gpu


def test_peer_plan_rejects_bad_destinations_and_binding():
    f = sq.builtin_fractal("sierpinski-triangle")
    p = sq.Squeeze(f, 10, rank=0, nranks=2, device=0)
    g = p.geometry
    sends = np.array([g.omega_lo, g.omega_lo + 1], dtype=np.uint64)
    p.halo_set_sends(sends)
    for bad in ([0, 1], [1, 2]):  # own rank, rank out of range
        with pytest.raises(sq.SqueezeError) as ei:
            p.halo_peer_plan(np.array(bad, dtype=np.uint32), np.zeros(2, dtype=np.uint64))
        assert ei.value.status == -6
    p.halo_peer_plan(np.array([1, 1], dtype=np.uint32), np.array([0, 1], dtype=np.uint64))
    buf = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(sq.SqueezeError):  # one pointer per rank
        p.halo_peer_bind(0, [buf.data_ptr()])
    p.halo_peer_bind(0, [0, buf.data_ptr()])
    p.halo_peer_select(0)
    with pytest.raises(sq.SqueezeError):  # parity 1 was never bound
        p.halo_peer_select(1)
    p.halo_set_sends(sends)  # drops the peer plan (it indexed the old send list)
    with pytest.raises(sq.SqueezeError):
        p.halo_peer_select(0)
    st = p.new_state()
    with pytest.raises(sq.SqueezeError):
        p.halo_peer_push(st, 0)


def test_run_host_rejects_sharded_context_before_copying():
    f = sq.builtin_fractal("sierpinski-triangle")
    p = sq.Squeeze(f, 8, rank=1, nranks=2, device=0)
    a, b = p.new_state(), p.new_state()
    h = torch.zeros(p.geometry.state_bytes, dtype=torch.uint8)
    with pytest.raises(sq.SqueezeError) as ei:
        p.run_host(h, a, b, 2)
    assert ei.value.status == -6


def test_binding_checks_device_tensors():
    p = sq.Squeeze(sq.builtin_fractal("sierpinski-triangle"), 8, device=0)
    a = p.new_state()
    with pytest.raises(sq.SqueezeError):  # int32 Ω would be read as int64 by the map kernel
        p.map_lambda(torch.zeros(8, dtype=torch.int32, device="cuda"))
    with pytest.raises(sq.SqueezeError):  # short state buffer
        p.step(a[:16], a)
    with pytest.raises(sq.SqueezeError):  # non-contiguous
        p.seed(torch.zeros(2 * p.geometry.state_bytes, dtype=torch.uint8, device="cuda")[::2])
    assert p.device_error() == 0
