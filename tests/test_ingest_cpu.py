"""MATPOWER / load-series ingest vs the reference's parse.

``tests/golden/ingest.npz`` (``tools/make_ingest_goldens.py``) holds the
input texts -- the reference's bundled ``pkg/data`` cases and load series
plus malformed / edge-case variants -- and the reference's results:
per-unit arrays, ``branch_admittance`` of every branch, ``validate_case``,
or the ``CaseError`` message (reference ``matpower.py:115-357``).  This
package's parser must reproduce every array bit for bit and every error
message verbatim.
"""

import json

import numpy as np
import pytest

from fixture_models import GOLDEN
from oracle.parity import bit_equal
from paper_2510_12897_b200 import CaseError, branch_admittance, parse_case, parse_load_series, validate_case
from paper_2510_12897_b200.casearrays import case_to_arrays

_Z = {}


def golden():
    if not _Z:
        with np.load(GOLDEN / "ingest.npz") as z:
            _Z.update({k: z[k] for k in z.files})
        _Z["index"] = json.loads(bytes(_Z["index_json"]).decode())
    return _Z


def _text(a) -> str:
    return bytes(np.asarray(a, dtype=np.uint8)).decode()


CASES = sorted(golden()["index"]["cases"])
SERIES = sorted(golden()["index"]["series"])


@pytest.mark.parametrize("label", CASES)
def test_parse_case_matches_reference(label):
    z = golden()
    want = z["index"]["cases"][label]
    text = _text(z[f"text_{label}"])
    if "error" in want:
        with pytest.raises(CaseError) as ei:
            parse_case(text, name=label)
        assert str(ei.value) == want["error"]
        return
    case = parse_case(text, name=label)
    assert case.name == want["name"]
    for k, a in case_to_arrays(case).items():
        ref = z[f"case_{label}_{k}"]
        assert a.shape == ref.shape and bit_equal(np.asarray(a, dtype=np.float64), ref), (label, k)
    assert validate_case(case) == want["validate"]
    adm = z[f"adm_{label}"]
    fields = want["admittance_fields"]
    for i, br in enumerate(case.branches):
        err = want["admittance_errors"][i]
        if err:
            with pytest.raises(CaseError) as ei:
                branch_admittance(br)
            assert str(ei.value) == err
            continue
        a = branch_admittance(br)
        got = np.array([getattr(a, f) for f in fields], dtype=np.float64)
        assert bit_equal(got, adm[i]), (label, i)


@pytest.mark.parametrize("label", SERIES)
def test_parse_load_series_matches_reference(label):
    z = golden()
    want = z["index"]["series"][label]
    text = _text(z[f"series_text_{label}"])
    if "error" in want:
        with pytest.raises(CaseError) as ei:
            parse_load_series(text, want["n_bus"], want["base_mva"])
        assert str(ei.value) == want["error"]
        return
    T, M = parse_load_series(text, want["n_bus"], want["base_mva"])
    assert T == want["T"]
    assert bit_equal(M, z[f"series_{label}"])


def test_parsed_case14_builds_the_golden_model():
    """The fixture model built from the parsed .m text equals the one built
    from the golden case arrays (same COO and bounds)."""
    from fixture_models import build, load

    from paper_2510_12897_b200 import opf_model

    z = golden()
    m_text = opf_model(parse_case(_text(z["text_case14"]), name="case14"), lower_to_gpu=False)[0]
    m_arr = build("case14_polar", lower_to_gpu=False)
    g = load("case14_polar")
    for a, b in ((m_text.plan.jac_rows, g["jac_rows"]), (m_text.plan.jac_cols, g["jac_cols"]),
                 (m_text.plan.hess_rows, g["hess_rows"]), (m_text.plan.hess_cols, g["hess_cols"]),
                 (m_text.lower, g["lower"]), (m_text.upper, g["upper"]), (m_text.start, g["start"])):
        assert np.array_equal(a, b)
    assert m_text.nvar == m_arr.nvar and m_text.ncon == m_arr.ncon
