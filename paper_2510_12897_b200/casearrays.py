"""CaseData <-> flat per-unit arrays (fixture and shard transport format)."""

from __future__ import annotations

import numpy as np

from .matpower import Branch, Bus, CaseData, Gen, Storage

_BUS = ("bus_id", "bus_type", "pd", "qd", "gs", "bs", "vmax", "vmin")
_GEN = ("bus_id", "pmin", "pmax", "qmin", "qmax", "status", "c2", "c1", "c0")
_BR = ("f_bus", "t_bus", "r", "x", "b_charging", "rate_a", "tap", "shift", "status", "angmin", "angmax")
_ST = ("bus_id", "energy_rating", "charge_rating", "discharge_rating", "eta_charge", "eta_discharge")
_INT = {"bus_id", "bus_type", "status", "f_bus", "t_bus"}


def _pack(items, names):
    return np.array([[float(getattr(it, n)) for n in names] for it in items], dtype=np.float64).reshape(
        len(items), len(names))


def _unpack(arr, names, cls):
    out = []
    for row in np.asarray(arr).reshape(-1, len(names)):
        kw = {n: (int(v) if n in _INT else float(v)) for n, v in zip(names, row)}
        out.append(cls(**kw))
    return out


def case_to_arrays(case: CaseData) -> dict:
    return {
        "name": np.frombuffer(case.name.encode(), dtype=np.uint8),
        "base_mva": np.float64(case.base_mva),
        "bus": _pack(case.buses, _BUS),
        "gen": _pack(case.gens, _GEN),
        "branch": _pack(case.branches, _BR),
        "storage": _pack(case.storage, _ST),
    }


def arrays_to_case(d: dict) -> CaseData:
    return CaseData(
        bytes(np.asarray(d["name"], dtype=np.uint8)).decode(),
        float(d["base_mva"]),
        _unpack(d["bus"], _BUS, Bus),
        _unpack(d["gen"], _GEN, Gen),
        _unpack(d["branch"], _BR, Branch),
        _unpack(d["storage"], _ST, Storage),
    )
