"""Custom combine operators (API extension, SURVEY 8(b) "Custom combine";
the reference's BinOpKind is closed, proj/include/mdh/mda.hpp:52, and its
JSON takes only pw:/ps: over + * min max - /, proj/src/json_io.cpp:58-64).
Host side only: parsing, validity and the registry (no GPU)."""
import json
import os

import pytest

from conftest import REPO
from oracle import refbind

SPEC = os.path.join(REPO, "specs", "extensions", "prl_max_prl.json")


def load(sizes=None):
    with open(SPEC) as f:
        j = json.load(f)
    if sizes:
        j["sizes"] = sizes
    return j


def test_max_prl_is_builtin():
    from paper_2405_05118_b200 import mdh
    ops = {o["name"]: o for o in mdh.combine_info()}
    m = ops["max_prl"]
    assert m["arity"] == 2 and m["assoc"] and m["comm"] and m["builtin"]
    assert m["identity"] == ["INT64_MIN", "INT64_MAX"]


def test_custom_operator_parses_and_lowers():
    from paper_2405_05118_b200 import mdh
    j = load([64, 4096])
    text = mdh.lowered(j, "B200")
    assert "pw:max_prl" in text
    cost, _ = mdh.simcost(j, "B200")
    assert cost > 0


def test_unknown_operator_is_rejected_with_the_reference_code():
    from paper_2405_05118_b200 import mdh
    j = load([64, 4096])
    j["combine"] = ["cc", "pw:no_such_op"]
    with pytest.raises(mdh.MdhError) as e:
        mdh.simcost(j, "B200")
    assert e.value.code == "UnknownOperator"


def test_arity_must_match_the_scalar_function():
    from paper_2405_05118_b200 import mdh
    j = load([64, 4096])
    j["outputs"] = j["outputs"][:1]
    j["scalar"] = j["scalar"].split(";")[0] + ";"
    with pytest.raises(mdh.MdhError) as e:
        mdh.simcost(j, "B200")
    assert e.value.code == "MixedIncompatibleOperators"


def test_mixing_custom_and_builtin_operators_is_not_an_md_hom():
    from paper_2405_05118_b200 import mdh
    j = load([64, 4096])
    j["dims"] = ["q", "r", "s"]
    j["sizes"] = [4, 8, 2]
    j["combine"] = ["cc", "pw:max_prl", "pw:max"]
    j["inputs"][1]["accesses"] = ["j + k, 0", "j, 1", "j, 2", "j, 3"]
    with pytest.raises(mdh.MdhError) as e:  # md_hom validity is checked before any device work
        mdh.Plan(j)
    assert e.value.code == "MixedIncompatibleOperators"


def test_user_registration_and_rules():
    from paper_2405_05118_b200 import mdh
    mdh.register_combine("argmin_lo", 2, "if (b0 < a0 || (b0 == a0 && b1 < a1)) { a0 = b0; a1 = b1; }",
                         identity=("INT64_MAX", "INT64_MAX"), description="lexicographic min")
    assert "argmin_lo" in {o["name"] for o in mdh.combine_info()}
    for bad in ("+", "max"):  # the reference's own operators cannot be redefined
        with pytest.raises(mdh.MdhError):
            mdh.register_combine(bad, 1, "a0 = b0;")
    with pytest.raises(mdh.MdhError):
        mdh.register_combine("max_prl", 2, "a0 = b0;")  # built-in
    mdh.register_combine("not_comm", 1, "a0 = b0;", comm=False)
    j = load([64, 4096])
    j["outputs"] = j["outputs"][:1]
    j["scalar"] = j["scalar"].split(";")[0] + ";"
    j["combine"] = ["cc", "pw:not_comm"]
    with pytest.raises(mdh.MdhError) as e:  # not associative+commutative: Lemma 2.9
        mdh.Plan(j)
    assert e.value.code == "MixedIncompatibleOperators"


@pytest.mark.skipif(not refbind.available(), reason="oracle/_ref not built")
def test_reference_rejects_the_extension():
    # the unmodified reference does not know the operator: this IS an extension
    with pytest.raises(refbind.RefError):
        refbind.reference_execute(json.dumps(load([4, 8])), [])
