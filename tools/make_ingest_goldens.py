"""Ingest goldens: the REFERENCE's MATPOWER / load-series parse.

Run in the build container (where /root/reference exists):

    python tools/make_ingest_goldens.py

For every bundled data file (``pkg/data/*.m``, ``case3_{pd,qd}.txt``) and a
set of malformed / edge-case variants of a small inline case (comments inside
blocks, trailing separators, ragged rows, missing blocks, unsupported cost
models, bad reference buses, dangling generators, zero taps, two-coefficient
costs, storage), it records the input text and the reference's result of
``parse_case`` (``matpower.py:164-275``) -- the per-unit arrays, every
``branch_admittance`` (115-129) and ``validate_case`` (283-331) -- or the
``CaseError`` message; likewise ``parse_load_series`` (334-357).  The inputs
are committed with the outputs (``tests/golden/ingest.npz``) so the test and
the GPU smoke test run without the reference.
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_DATA = Path("/root/reference/pkg/data")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "ingest.npz"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import simdnlp as ref  # noqa: E402

from make_goldens import our_case_from_ref  # noqa: E402
from paper_2510_12897_b200.casearrays import case_to_arrays  # noqa: E402

SMALL = """
function mpc = small
mpc.version = '2';
mpc.baseMVA = 100;
%% bus data
mpc.bus = [
    1 3 90.0 30.0 5.0 2.0 1 1.0 0.0 230 1 1.1 0.9;
    2 2 50.0 10.0 0.0 0.0 1 1.0 0.0 230 1 1.1 0.9;
    3 1 20.0 -4.0 0.0 19.0 1 1.0 0.0 230 1 1.05 0.95;
];
mpc.gen = [
    1 10 0 30 -30 1.0 100 1 40 5;
    2 20 0 60 -60 1.0 100 1 80 0;
];
mpc.gencost = [
    2 0 0 3 0.11 5 0;
    2 0 0 3 0.02 12 150;
];
mpc.branch = [
    1 2 0.01938 0.05917 0.0528 130 0 0 0 0 1 -30 30;
    2 3 0.0 0.2 0.0 0 0 0 0.98 2.5 1 -60 60;
    1 3 0.05 0.22 0.04 90 0 0 1.02 0 0 -360 360;
];
"""


def variants():
    v = {"small": SMALL}
    v["comments_separators"] = SMALL.replace(
        "    2 3 0.0 0.2 0.0 0 0 0 0.98 2.5 1 -60 60;",
        "\n  % a comment inside the block\n    2 3 0.0 0.2 0.0 0 0 0 0.98 2.5 1 -60 60 ; \n\n")
    v["two_coefficient_cost"] = SMALL.replace("2 0 0 3 0.02 12 150", "2 0 0 2 12 150").replace(
        "2 0 0 3 0.11 5 0", "2 0 0 2 5 0")
    v["missing_gencost"] = SMALL.replace("mpc.gencost", "mpc.ignored")
    v["missing_branch"] = SMALL.replace("mpc.branch", "mpc.nobranch")
    v["missing_basemva"] = SMALL.replace("mpc.baseMVA = 100;", "")
    v["negative_basemva"] = SMALL.replace("mpc.baseMVA = 100;", "mpc.baseMVA = -5;")
    v["ragged"] = SMALL.replace("2 2 50.0 10.0 0.0 0.0 1 1.0 0.0 230 1 1.1 0.9;", "2 2 50.0;")
    v["piecewise_cost"] = SMALL.replace("2 0 0 3 0.11 5 0", "1 0 0 2 0 0 1 1").replace(
        "2 0 0 3 0.02 12 150", "1 0 0 2 0 0 2 2")
    v["quartic_cost"] = SMALL.replace("2 0 0 3 0.11 5 0", "2 0 0 4 1 0.11 5 0").replace(
        "2 0 0 3 0.02 12 150", "2 0 0 4 0 0.02 12 150")
    v["ragged_cost_rows"] = SMALL.replace("2 0 0 3 0.11 5 0", "2 0 0 3 0.11")
    v["short_cost_row"] = SMALL.replace("2 0 0 3 0.11 5 0", "2 0 0 3 0.11 5").replace(
        "2 0 0 3 0.02 12 150", "2 0 0 3 0.02 12")
    v["non_numeric"] = SMALL.replace("0.01938", "zap")
    v["no_reference_bus"] = SMALL.replace("1 3 90.0", "1 1 90.0")
    v["two_reference_buses"] = SMALL.replace("2 2 50.0", "2 3 50.0")
    v["dangling_generator"] = SMALL.replace("mpc.gen = [\n    1 10", "mpc.gen = [\n    99 10")
    v["dangling_branch"] = SMALL.replace("1 3 0.05 0.22", "1 7 0.05 0.22")
    v["short_bus_rows"] = SMALL.replace("1 1.1 0.9;\n    2 2", "1 1.1;\n    2 2").replace(
        "1 1.1 0.9;\n    3 1", "1 1.1;\n    3 1").replace("1 1.05 0.95;", "1 1.05;")
    v["gen_cost_count_mismatch"] = SMALL.replace("    2 0 0 3 0.02 12 150;\n", "")
    v["empty_gen"] = SMALL.replace("    1 10 0 30 -30 1.0 100 1 40 5;\n    2 20 0 60 -60 1.0 100 1 80 0;\n", "")
    v["vmin_above_vmax"] = SMALL.replace("1 1.05 0.95;", "1 0.9 0.95;")
    v["degenerate_branch"] = SMALL.replace("1 2 0.01938 0.05917", "1 2 0.0 0.0")
    v["storage"] = SMALL + "\nmpc.storage = [\n    3 2.0 0.5 0.6 0.95 0.9;\n];\n"
    v["storage_bad_columns"] = SMALL + "\nmpc.storage = [\n    3 2.0 0.5;\n];\n"
    return v


def load_series_inputs():
    v = {}
    for n in ("case3_pd.txt", "case3_qd.txt"):
        v[n] = ((REF_DATA / n).read_text(), 3, 100.0)
    v["uniform"] = ("100 100 100\n100 100 100\n", 3, 100.0)
    v["single_row"] = ("10 20 30", 3, 100.0)
    v["comments_blank"] = ("% header\n\n10 20 30\n  40 50 60  \n", 3, 50.0)
    v["wrong_columns"] = ("1 2\n", 3, 100.0)
    v["non_numeric"] = ("1 2 x\n", 3, 100.0)
    v["empty"] = ("% only comments\n", 3, 100.0)
    return v


def text_arr(s: str) -> np.ndarray:
    return np.frombuffer(s.encode(), dtype=np.uint8)


def main():
    arrays = {}
    index = {"cases": {}, "series": {}}
    inputs = {p.stem: p.read_text() for p in sorted(REF_DATA.glob("*.m"))}
    inputs.update(variants())
    for label, text in inputs.items():
        arrays[f"text_{label}"] = text_arr(text)
        try:
            case = ref.parse_case(text, name=label)
        except ref.CaseError as e:
            index["cases"][label] = {"error": str(e)}
            continue
        ours = our_case_from_ref(case)
        for k, a in case_to_arrays(ours).items():
            arrays[f"case_{label}_{k}"] = a
        adm = []
        adm_err = []
        for br in case.branches:
            try:
                a = ref.branch_admittance(br)
                adm.append([getattr(a, f.name) for f in dataclasses.fields(a)])
                adm_err.append("")
            except ref.CaseError as e:
                adm.append([np.nan] * 9)
                adm_err.append(str(e))
        arrays[f"adm_{label}"] = np.array(adm, dtype=np.float64).reshape(len(case.branches), -1)
        index["cases"][label] = {"validate": ref.validate_case(case), "admittance_errors": adm_err,
                                 "name": case.name,
                                 "admittance_fields": [f.name for f in dataclasses.fields(ref.BranchAdmittance)]}
    for label, (text, nb, base) in load_series_inputs().items():
        arrays[f"series_text_{label}"] = text_arr(text)
        try:
            T, M = ref.parse_load_series(text, nb, base)
            arrays[f"series_{label}"] = M
            index["series"][label] = {"n_bus": nb, "base_mva": base, "T": T}
        except ref.CaseError as e:
            index["series"][label] = {"n_bus": nb, "base_mva": base, "error": str(e)}
    arrays["index_json"] = text_arr(json.dumps(index))
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(index['cases'])} case inputs "
          f"({sum('error' in v for v in index['cases'].values())} errors), {len(index['series'])} load series")


if __name__ == "__main__":
    main()
