"""Rebuild the golden fixtures with this package (no reference needed)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2510_12897_b200 import opf as P
from paper_2510_12897_b200.casearrays import arrays_to_case
from paper_2510_12897_b200.core import DataTable, ModelCore
from paper_2510_12897_b200.expressions import cos, exp, field, log, sin, sqrt
from paper_2510_12897_b200.problems import luksan_vlcek_model

GOLDEN = Path(__file__).resolve().parent / "golden"
INDEX = json.loads((GOLDEN / "index.json").read_text())
NAMES = sorted(INDEX)


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def custom_model(which: str, lower_to_gpu: bool):
    core = ModelCore()
    if which == "product":
        x = core.add_variable(2)
        core.add_objective(x["a"] * x["b"], DataTable({"a": np.array([0]), "b": np.array([1])}))
    elif which == "dupvar":
        x = core.add_variable(3)
        core.add_objective(x["a"] * x["b"] + x["a"] ** 3,
                           DataTable({"a": np.array([0, 1, 2]), "b": np.array([0, 2, 2])}))
    elif which == "allops":
        x = core.add_variable(2, lower=[0.2, 0.3], upper=[3.0, 3.0], start=1.0)
        t = DataTable({"i": np.array([0, 1, 0]), "j": np.array([1, 0, 1]), "w": np.array([0.7, 1.3, 2.1])})
        kern = (sin(x["i"]) + cos(x["j"]) * exp(x["i"]) - log(x["j"]) / sqrt(x["i"])
                + x["i"] ** 3 - (-x["j"]) + field("w") ** x["i"] + x["i"] / x["j"])
        core.add_objective(kern, t)
        core.add_constraint(kern * x["j"] - 2.0 * x["i"] ** -2, t)
    elif which == "augments":
        x = core.add_variable(4, lower=0.1, upper=2.0, start=1.0)
        base = core.add_constraint(x["i"] ** 2 - field("c"),
                                   DataTable({"i": np.array([0, 1, 2]), "c": np.array([1.0, 2.0, 3.0])}))
        core.modify_constraint(base, 2.0 * x["k"] * x["i"], DataTable(
            {"k": np.array([3, 3, 0, 1]), "i": np.array([0, 1, 1, 2]), "row": np.array([0, 1, 1, 2])}))
        core.modify_constraint(base, -x["k"], DataTable({"k": np.array([2, 2]), "row": np.array([2, 0])}))
        core.add_constraint(x["i"] * 0.0 + x["k"] - x["k"],
                            DataTable({"i": np.array([0, 1]), "k": np.array([2, 3])}))
        core.add_objective(x["a"] ** x["b"], DataTable({"a": np.array([0, 1]), "b": np.array([1, 2])}))
    else:
        raise KeyError(which)
    return core.compile(lower_to_gpu=lower_to_gpu)


def build(name: str, lower_to_gpu: bool = False, data: dict | None = None):
    spec = INDEX[name]
    data = data if data is not None else load(name)
    kind = spec["kind"]
    if kind in ("opf", "mpopf"):
        case = arrays_to_case({k[5:]: v for k, v in data.items() if k.startswith("case_")})
        if kind == "opf":
            return P.opf_model(case, form=spec["form"], lower_to_gpu=lower_to_gpu)[0]
        return P.mpopf_model(case, np.array(spec["curve"]), spec["car"], spec["complementarity"],
                             form=spec["form"], lower_to_gpu=lower_to_gpu)[0]
    if kind == "lv":
        return luksan_vlcek_model(spec["n"], lower_to_gpu=lower_to_gpu)[0]
    return custom_model(spec["which"], lower_to_gpu)
