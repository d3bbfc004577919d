"""The C-ABI library loads and exports every symbol include/flern.h declares (CPU-only), and
refuses to run without an sm_100 GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flern.h")
LIB = os.path.join(ROOT, "paper_2311_02781_b200", "lib", "libflern.so")


def declared_functions():
    src = open(HEADER).read()
    return re.findall(r"FLERN_API\s+[\w\s\*]+?\b(flern_\w+)\s*\(", src)


def test_header_declares_the_boundary():
    fns = declared_functions()
    for need in ("flern_load_table", "flern_load_model", "flern_build_hashtable", "flern_run_query",
                 "flern_create", "flern_destroy", "flern_last_error"):
        assert need in fns


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_2311_02781_b200 import flern as F
    assert set(F.EXPORTED) == set(declared_functions())
    for f in F.EXPORTED:
        assert callable(getattr(F, f))


def test_version_and_launch_count():
    from paper_2311_02781_b200 import flern as F
    assert "sm_100a" in F.flern_version()
    assert F.flern_query_launches() == 1


def test_kernels_are_sm100a_tcgen05():
    """The library's SASS holds tcgen05 MMAs (UTCHMMA, incl. the CTA-pair form) and TMEM loads (LDTM):
    the MLP runs on the 5th-generation tensor cores, not mma.sync (HMMA); operands arrive by TMA
    (UTMALDG) and bulk copies (UBLKCP)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "LDTM" in sass
    assert " HMMA" not in sass
    # the wide kernel: CTA-pair MMAs (cta_group::2) fed by tensor-map TMA
    assert "UTCHMMA.2CTA" in sass and "UTMALDG" in sass
    # the fact-column loader and the narrow kernels' operand copies: bulk async copies
    assert "UBLKCP" in sass


def test_no_gpu_means_error_not_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2311_02781_b200 import flern as F
    with pytest.raises(F.FlernError):
        F.flern_create(0)


def test_missing_library_fails_loudly():
    """Without the built library the binding refuses to import: there is no fallback path."""
    import subprocess
    import sys
    env = dict(os.environ, FLERN_LIB="libflern_does_not_exist.so")
    r = subprocess.run([sys.executable, "-c", "import paper_2311_02781_b200.flern"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "libflern_does_not_exist.so is missing" in r.stderr
