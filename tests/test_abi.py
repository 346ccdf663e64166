"""CPU checks of the C ABI: libnb.so loads without a GPU and exports every
function include/nb.h declares; host-only entry points answer correctly."""
import ctypes as C
import os
import re

import pytest

import paper_2310_06822_b200 as nb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "nb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_five_hot_path_calls():
    fns = declared_functions()
    for f in ["nb_encode", "nb_forward", "nb_train_step", "nb_calibrate", "nb_score"]:
        assert f in fns


def test_library_exports_every_declared_symbol():
    L = C.CDLL(nb.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert set(declared_functions()) == set(nb.SIGNATURES), \
        set(declared_functions()) ^ set(nb.SIGNATURES)


def test_host_only_calls():
    L = nb.lib()
    assert L.nb_record_floats(nb.POINT, 3) == 3
    assert L.nb_record_floats(nb.RAY, 3) == 6
    assert L.nb_record_floats(nb.POINT, 4) == 4
    assert L.nb_record_floats(nb.RAY, 4) == 8      # 4D rays: (origin, direction) in (x, y, z, t) (R48)
    assert L.nb_record_floats(nb.BOX, 5) == -1
    assert nb.Desc("point", 3, 50, 2, precision="fp32").num_params == 2801
    assert nb.Desc("point", 4, 128, 6, (2, 4)).num_params == 83587
    assert nb.alpha(0, 200) == 1.0 and nb.alpha(199, 200) == 1000.0
    assert L.nb_status_string(5) == b"no positive labels (tau = +inf)"


def test_invalid_desc_rejected_without_gpu():
    d = nb.Desc("ray", 5, 64, 4).to_c()          # no 5D records
    assert nb.lib().nb_num_params(C.byref(d)) == -1
    assert nb.Desc("ray", 4, 64, 4).num_params == (8 + 1) * 64 + 3 * 65 * 64 + 65  # 4D ray: 8 inputs (R48)
    h = C.c_void_p()
    assert nb.lib().nb_model_create(C.byref(d), 0, C.byref(h)) == 1  # NB_E_ARG


def test_header_is_plain_c99(tmp_path):
    """include/nb.h is a C ABI: it compiles as strict C99 (no C++ or torch types)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    src = tmp_path / "use.c"
    src.write_text('#include "nb.h"\nint main(void) { nb_desc d = {0}; nb_counts c; nb_schedule s;\n'
                   '  (void)d; (void)c; (void)s; return nb_record_floats(NB_POINT, 3) == 3 ? 0 : 1; }\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                        os.path.join(ROOT, "include"), "-c", str(src), "-o", str(tmp_path / "use.o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
