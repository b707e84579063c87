"""The host-staged collectives behind rlra_comm_create_host (csrc/dist.cu
LocalGroup), exercised on the CPU: the C-ABI hands out the group's function
pointers, which need no GPU.  Ranks are Python threads calling them through
ctypes (the GIL is released during foreign calls)."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_1502_05366_b200 as R


def _fns(group, rank):
    hc = group.collectives(rank).struct()
    ar = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t)(hc.allreduce_sum)
    ag = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t)(hc.allgather)
    acq = C.CFUNCTYPE(None, C.c_void_p)(hc.gpu_acquire)
    rel = C.CFUNCTYPE(None, C.c_void_p)(hc.gpu_release)
    return hc.user, ar, ag, acq, rel


def _run(world, body, timeout=60.0):
    g = R.LocalGroup(world, timeout_s=timeout)
    out, err = [None] * world, [None] * world

    def th(r):
        try:
            out[r] = body(r, *_fns(g, r))
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=th, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not any(t.is_alive() for t in ts)
    g.close()
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_allreduce_sums_in_rank_order_identically_on_every_rank(world):
    rs = np.random.default_rng(world)
    data = [rs.standard_normal(1000) * 10.0 ** rs.integers(-8, 8, 1000) for _ in range(world)]

    def body(r, user, ar, ag, acq, rel):
        buf = data[r].copy()
        assert ar(user, buf.ctypes.data_as(C.POINTER(C.c_double)), buf.size) == 0
        return buf

    res = _run(world, body)
    want = np.zeros(1000)
    for d in data:  # rank order, left to right
        want = want + d
    for b in res:
        assert np.array_equal(b, want)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_allgather_places_rank_r_at_offset_r(world):
    def body(r, user, ar, ag, acq, rel):
        send = np.full(7, float(r)) + np.arange(7) * 0.5
        recv = np.zeros(7 * world)
        assert ag(user, send.ctypes.data_as(C.POINTER(C.c_double)), recv.ctypes.data_as(C.POINTER(C.c_double)),
                  7) == 0
        return recv

    for recv in _run(world, body):
        for r in range(world):
            assert np.array_equal(recv[7 * r:7 * r + 7], np.full(7, float(r)) + np.arange(7) * 0.5)


def test_mismatched_counts_fail_on_every_rank():
    def body(r, user, ar, ag, acq, rel):
        buf = np.ones(10 + r)
        return ar(user, buf.ctypes.data_as(C.POINTER(C.c_double)), buf.size)

    assert all(rc != 0 for rc in _run(2, body))


def test_a_missing_rank_times_out_instead_of_hanging():
    def body(r, user, ar, ag, acq, rel):
        if r == 1:
            return 0  # never joins the collective
        buf = np.ones(4)
        return ar(user, buf.ctypes.data_as(C.POINTER(C.c_double)), buf.size)

    res = _run(2, body, timeout=1.0)
    assert res[0] != 0


def test_gpu_token_is_exclusive():
    inside = []
    lock = threading.Lock()

    def body(r, user, ar, ag, acq, rel):
        for _ in range(50):
            acq(user)
            with lock:
                inside.append(1)
                assert sum(inside) == 1
            with lock:
                inside.pop()
            rel(user)
        return 0

    _run(4, body)
