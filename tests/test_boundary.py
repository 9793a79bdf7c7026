"""CPU-side checks of the drop-in boundary: the C-ABI library builds for
sm_100a, loads without a GPU, and exports every entry point that
include/ttround_b200.h declares; status codes mirror the reference Errc order."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ttround_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:ttr_status|const char\*)\s+(ttr_\w+)\s*\(", text, re.M)))


def test_header_declares_the_hot_path_entry_points():
    syms = declared_symbols()
    for s in ["ttr_round_fixed_krp", "ttr_round_adaptive_krp", "ttr_round_deterministic_tol",
              "ttr_round_deterministic_ranks", "ttr_estimate_norm_krp", "ttr_tt_upload", "ttr_tt_download",
              "ttr_norm_exact", "ttr_relative_error", "ttr_krp_partial_contractions", "ttr_plan_fixed_krp", "ttr_plan_fixed_krp_host", "ttr_round_sum_adaptive_krp", "ttr_compression_pass", "ttr_round_rand_orth_tt", "ttr_tt_read_ttf1", "ttr_tt_write_ttf1"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_2511_03598_b200 as P
    lib = P.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a_code():
    import paper_2511_03598_b200 as P
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_codes_mirror_reference_errc_order():
    """types.hpp:15-31 order; the header assigns 1 + index."""
    import paper_2511_03598_b200 as P
    text = open(os.path.join(ROOT, "include", "ttround_b200.h")).read()
    names = ["RANK_CHAIN_MISMATCH", "BOUNDARY_RANK_NOT_ONE", "EMPTY_CORE_LIST", "INDEX_OUT_OF_RANGE",
             "DENSE_TOO_LARGE", "MODE_SIZE_MISMATCH", "EMPTY_TERM_LIST", "INVALID_RANK_CHAIN", "SVD_FAILURE",
             "INVALID_RANKS", "NOT_LEFT_ORTHOGONAL", "INVALID_GRID", "BREAKDOWN", "INVALID_ARGUMENT", "IO"]
    for i, n in enumerate(names):
        assert re.search(rf"TTR_ERR_{n}\s*=\s*{i + 1}\b", text), n
    assert P.ERRC_NAMES[9] == "InvalidRanks"


def test_no_device_fails_loudly():
    """Without a GPU the product raises instead of silently computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2511_03598_b200 as P
    with pytest.raises(P.TTRoundError) as e:
        P.Context(0)
    assert e.value.code == "NoDevice"


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2511_03598_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "py_oracle" not in text and "ttr_oracle" not in text, f


def _build_wrapper_smoke(tmp_path):
    import paper_2511_03598_b200 as P
    exe = str(tmp_path / "wrapper_smoke")
    libdir = os.path.dirname(P.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "wrapper_smoke.cpp"), "-L", libdir, "-lttround_b200",
           f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_wrapper_compiles_and_links(tmp_path):
    """include/ttround_b200/ttround.hpp: the reference-shaped C++ API builds against the C ABI."""
    assert os.path.exists(_build_wrapper_smoke(tmp_path))


@pytest.mark.gpu
def test_cpp_wrapper_runs_on_device(tmp_path):
    exe = _build_wrapper_smoke(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "wrapper ok" in out.stdout


def _build_dropin(tmp_path):
    import paper_2511_03598_b200 as P
    exe = str(tmp_path / "dropin_vs_oracle")
    libdir = os.path.dirname(P.LIB_PATH)
    odir = os.path.join(ROOT, "oracle", "_build")
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "dropin_vs_oracle.cpp"), "-L", libdir, "-lttround_b200",
           "-L", odir, "-lttr_oracle", f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{odir}", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_dropin_vs_oracle_compiles_and_links(tmp_path):
    """tests/cpp/dropin_vs_oracle.cpp (every mirrored entry point vs the oracle) builds."""
    assert os.path.exists(_build_dropin(tmp_path))


@pytest.mark.gpu
def test_dropin_vs_oracle_runs_on_device(tmp_path):
    """The C++ drop-in layer on the device equals the oracle entry point by entry point:
    Core/TTTensor(vector<Core>), random_gaussian_tt (bitwise), dot, norm_exact, formal_sum,
    scaled, GaussianStream/draw_gaussian_factors/append_gaussian_columns (bitwise, reference
    stream), krp_partial_contractions_rl, append_krp_contractions, generate_residual_sketch,
    residual_norm_estimate, round_fixed_krp / round_adaptive_krp / round_deterministic /
    estimate_norm_krp (reference stream), build_cookie_problem / apply_operator / tt_gmres, and
    the constructor's error kinds."""
    exe = _build_dropin(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dropin ok" in out.stdout
