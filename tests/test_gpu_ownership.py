"""Write ownership (SPEC.md:350's debug ownership map, on the GPU): the
DCONV_DEBUG_OWNERSHIP build counts every conv output store; every case of
tests/_ownership_cases.py must write each element of its output view exactly
once and nothing outside it.  Runs in a subprocess because the debug library
replaces the product one (DCONV_LIB)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OWN = os.path.join(ROOT, "paper_1809_10170_b200", "libdconv_b200_own.so")

pytestmark = pytest.mark.gpu


def test_every_output_element_written_exactly_once():
    assert os.path.exists(OWN), "build the ownership library: make -C paper_1809_10170_b200/csrc own"
    env = dict(os.environ, DCONV_LIB=OWN)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_ownership_cases.py")],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "every output element written exactly once" in r.stdout
    print(r.stdout.splitlines()[0])


def test_product_build_has_no_ownership_hook():
    """The product library compiles the hook out: the call is refused."""
    from paper_1809_10170_b200 import _abi
    if "_own" in _abi.LIB_PATH:
        pytest.skip("running against the debug build")
    assert _abi.lib().dconv_debug_set_ownership(None, None, 0) == _abi.EUNSUPPORTED
