"""di_set_option / di_get_option (include/di.h): every knob of the library, no environment variable.
CPU-only: the calls touch no device."""
import pytest

di = pytest.importorskip("paper_1204_6255_b200")

DEFAULTS = {"red_hint": 1, "push_occ": 4, "auto_ratio": 0.35, "stripes": 0, "hot_acc": 1,
            "repl_share": 0.0005, "cold_bins": -1, "cold_tier": 0, "cold_shift": 0,
            "cycle_grid_div": 1, "cycle_times": 0, "p2p": 1, "p2p_force": 0, "build_trace": 0,
            "remote_compact": 1, "remote_tier": 0, "long_lanes": 1, "row_sort": 0, "line_spread": 16,
            "warm": -1, "warm_flush": 0, "warm_shift": 0,
            "dist_parts": 1}


def test_defaults_documented_and_settable():
    header = open(__import__("os").path.join(__import__("os").path.dirname(__file__), "..", "include",
                                             "di.h")).read()
    for name, v in DEFAULTS.items():
        assert di.get_option(name) == pytest.approx(v), name
        assert f'"{name}"' in header, name            # every option is documented in di.h
        with di.option(name, v):
            assert di.get_option(name) == pytest.approx(v)
    with di.option("cold_bins", 1):
        assert di.get_option("cold_bins") == 1
    assert di.get_option("cold_bins") == -1            # restored


@pytest.mark.parametrize("name,value", [("nope", 1), ("red_hint", 2), ("push_occ", 0), ("cold_bins", 3),
                                        ("line_spread", 3), ("stripes", 1.5), ("auto_ratio", float("nan")),
                                        ("warm", -2), ("warm", 70000), ("dist_parts", 0),
                                        ("dist_parts", 65), ("warm_shift", 31)])
def test_bad_options_refused(name, value):
    with pytest.raises(di.DIError) as ei:
        di.set_option(name, value)
    assert ei.value.status == di.DI_EINVAL
    with pytest.raises(di.DIError):
        di.get_option("nope")


def test_library_reads_no_environment():
    import os
    src = os.path.join(os.path.dirname(__file__), "..", "paper_1204_6255_b200", "csrc")
    for f in os.listdir(src):
        if f.endswith((".cu", ".cuh")):
            assert "getenv" not in open(os.path.join(src, f)).read(), f
