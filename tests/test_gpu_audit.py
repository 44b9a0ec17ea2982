"""EREW shadow-writer audit:
the partition's kernels in the debug build libpp_audit.so count every key
store per phase; tests/erew_audit_run.py asserts each key is written at most
once by the group kernel and at most once by the cleanup, the group kernel
writes exactly its full lines, the cleanup exactly the 2M misplaced keys, and
the result is the oracle's partition.  Run in a subprocess so that the audit
library, not libpp.so, is the one loaded (PP_LIB_PATH)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AUDIT_LIB = os.path.join(ROOT, "paper_2004_12532_b200", "libpp_audit.so")


@pytest.mark.gpu
def test_erew_shadow_writer_audit():
    assert os.path.exists(AUDIT_LIB), "libpp_audit.so missing: run __graft_entry__.build()"
    env = dict(os.environ, PP_LIB_PATH=AUDIT_LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "erew_audit_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "EREW AUDIT OK" in r.stdout, (r.stdout[-3000:], r.stderr[-3000:])


def test_product_library_has_no_audit():
    """The product library rejects pp_audit_set (the counters exist only in
    the debug build, so libpp.so keeps its no-atomics SASS)."""
    import paper_2004_12532_b200 as pp
    lib = pp.load(build_if_missing=False)
    assert lib.pp_audit_set(None, None, 0, 0) == 1  # PP_E_INVAL
