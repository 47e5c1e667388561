"""Host logic of the in-place page locking of reused numpy buffers
(``autodiff._HostPins``), against a stand-in for ``libexa``'s
``exa_host_register`` / ``exa_host_unregister`` (no GPU needed)."""

import gc

import numpy as np
import pytest

from paper_2510_12897_b200.autodiff import _HostPins


class FakeLib:
    def __init__(self, fail=False):
        self.live, self.calls, self.fail = {}, [], fail

    def exa_host_register(self, ptr, nbytes):
        self.calls.append(("reg", ptr.value, nbytes))
        if self.fail:
            return 1
        self.live[ptr.value] = nbytes
        return 0

    def exa_host_unregister(self, ptr):
        self.calls.append(("unreg", ptr.value))
        assert self.live.pop(ptr.value, None) is not None, "unregister of a range never registered"
        return 0


def _pins():
    p = _HostPins()
    p.enabled = True
    return p


def test_locked_on_second_use_and_released_on_free():
    pins, lib = _pins(), FakeLib()
    a = np.empty(pins.MIN_BYTES // 8)
    pins.note(lib, a)
    assert not lib.live and not pins.locked(a)
    pins.note(lib, a)
    assert lib.live == {a.ctypes.data: a.nbytes} and pins.locked(a)
    pins.note(lib, a)  # already locked: no second registration
    assert len(lib.calls) == 1
    del a
    gc.collect()
    assert not lib.live and not pins._spans and pins._bytes == 0


def test_small_and_one_shot_arrays_are_not_locked():
    pins, lib = _pins(), FakeLib()
    small = np.empty(pins.MIN_BYTES // 8 - 1)
    for _ in range(3):
        pins.note(lib, small)
    for _ in range(3):
        pins.note(lib, np.empty(pins.MIN_BYTES // 8))  # a new array every call
    assert not lib.calls and not pins._spans


def test_views_lock_their_owner_once():
    pins, lib = _pins(), FakeLib()
    owner = np.empty(3 * pins.MIN_BYTES // 8)
    n = pins.MIN_BYTES // 8
    v1, v2 = owner[:n], owner[n:2 * n]
    pins.note(lib, v1)
    pins.note(lib, v2)
    assert lib.live == {owner.ctypes.data: owner.nbytes}
    assert pins.locked(v1) and pins.locked(v2) and pins.locked(owner)
    del v1, v2, owner
    gc.collect()
    assert not lib.live


def test_small_view_of_a_large_owner_is_skipped():
    pins, lib = _pins(), FakeLib()
    pins.SLACK_BYTES = 0
    owner = np.empty(8 * pins.MIN_BYTES // 8)
    small = owner[:pins.MIN_BYTES // 8]
    for _ in range(3):
        pins.note(lib, small)
    assert not lib.calls
    big = owner[pins.MIN_BYTES // 8:]
    pins.note(lib, big)
    pins.note(lib, big)
    assert lib.live == {owner.ctypes.data: owner.nbytes} and pins.locked(small)


def test_arrays_not_owning_memory_are_skipped():
    pins, lib = _pins(), FakeLib()
    buf = bytearray(pins.MIN_BYTES)
    a = np.frombuffer(buf, dtype=np.float64)  # memory owned by a non-numpy object
    for _ in range(3):
        pins.note(lib, a)
    assert not lib.calls


def test_overlapping_bytes_and_byte_cap_are_refused():
    pins, lib = _pins(), FakeLib()
    a = np.empty(pins.MIN_BYTES // 8)
    pins.note(lib, a)
    pins.note(lib, a)
    assert pins.locked(a)
    fin = pins._spans[id(a)][2]
    # a range sharing bytes with a locked one is left pageable (sharing pages is fine)
    b = np.empty(pins.MIN_BYTES // 8)
    key = 12345
    pins._spans[key] = (b.ctypes.data + b.nbytes - 8, b.ctypes.data + b.nbytes + 8, fin)
    pins.note(lib, b)
    pins.note(lib, b)
    assert not pins.locked(b)
    pins._spans[key] = (b.ctypes.data + b.nbytes, b.ctypes.data + b.nbytes + 4096, fin)
    pins._seen.clear()
    pins.MAX_BYTES = pins._bytes + b.nbytes - 1
    pins.note(lib, b)
    pins.note(lib, b)
    assert not pins.locked(b), "the total lock cap must hold"
    pins.MAX_BYTES = 1 << 40
    pins.note(lib, b)
    assert pins.locked(b), "a neighbour on the same page does not block the lock"
    del pins._spans[key]


def test_failed_registration_leaves_the_array_pageable():
    pins, lib = _pins(), FakeLib(fail=True)
    a = np.empty(pins.MIN_BYTES // 8)
    for _ in range(4):
        pins.note(lib, a)
    assert not pins.locked(a) and not pins._spans
    assert len(lib.calls) == 1, "a refused array is not retried"
    key = id(a)
    del a
    gc.collect()
    assert key not in pins._refused and key not in pins._seen


def test_locked_memory_cannot_move():
    """A locked array's memory cannot be re-allocated under the lock: numpy
    refuses ndarray.resize on an array that is weakly referenced (the
    finalizer that drops the lock)."""
    pins, lib = _pins(), FakeLib()
    a = np.empty(pins.MIN_BYTES // 8)
    pins.note(lib, a)
    pins.note(lib, a)
    with pytest.raises(ValueError):
        a.resize(8 * a.size, refcheck=False)
    assert lib.live == {a.ctypes.data: a.nbytes}


def test_disabled():
    pins, lib = _pins(), FakeLib()
    pins.enabled = False
    a = np.empty(pins.MIN_BYTES // 8)
    for _ in range(3):
        pins.note(lib, a)
    assert not lib.calls
