"""The reference's own test suite, run against this package's drop-in.

oracle/vendor_ref.py copies the reference package and its tests (unmodified)
into oracle/_ref/.  Here those test modules run in a pytest subprocess with
`framekv` = this package for every hot-path name (tests/conformance/
framekv_alias.py: numpy facade over the GPU kernels) and the vendored
reference for the rest.  No assertion of the reference tests is relaxed or
skipped; test_cli.py (needs matplotlib, absent from the image) is the only
module left out.
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
FILES = ["test_kvmodel.py", "test_layout.py", "test_rangecoder.py", "test_codec.py",
         "test_container.py", "test_fetchsim.py", "test_netstore.py", "test_scheduler.py",
         "test_acceptance.py"]
# the hot-path tests VERDICT r01 names (reference file:line ranges)
HOT = {
    "test_kvmodel.py": ["test_quantize_unit_range_oracle", "test_quantize_asymmetric_group_oracle",
                        "test_quantize_all_zero_group_scale_one", "test_quantize_rounds_half_to_even",
                        "test_quantize_validates_group_size", "test_dequantize_error_bound",
                        "test_paged_memory_accounting", "test_paged_memory_write_conflict",
                        "test_paged_memory_free_then_rewrite"],
    "test_fetchsim.py": ["test_restore_stream_matches_chunk_wise"],
    "test_acceptance.py": ["test_codec_lossless_on_random_sequences_and_all_tilings",
                           "test_loopback_fetch_restores_chunk_bitexact",
                           "test_framewise_restore_peak_at_most_tenth_of_chunkwise"],
}


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests", "conformance"),
                                         env.get("PYTHONPATH", "")])
    env["NUMBA_CACHE_DIR"] = "/tmp/numba_cache_framekv_ref"
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                               reason="oracle/_ref not vendored (python -m oracle.vendor_ref)")


@needs_ref
def test_alias_composition():
    """CPU: the alias takes exactly the HOT_PATH names from this package."""
    code = ("import framekv_alias, json; t = framekv_alias.build_alias(); import framekv, "
            "paper_2602_09725_b200.compat as c, framekv_ref.scheduler as rs; "
            "assert framekv.kvmodel.quantize is c.kvmodel.quantize; "
            "assert framekv.fetchsim.restore_stream is c.fetchsim.restore_stream; "
            "assert framekv.scheduler.run_trace is rs.run_trace; "
            "assert framekv.fetchsim.simulate_fetch.__module__ == 'framekv_ref.fetchsim'; "
            "print(json.dumps(t))")
    out = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    taken = json.loads(out.stdout.strip().splitlines()[-1])
    assert "restore_stream" in taken["fetchsim"] and "live_fetch_pipeline" in taken["netstore"]


@pytest.mark.gpu
@needs_ref
def test_reference_suite_through_drop_in(tmp_path):
    xml = tmp_path / "ref.xml"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "framekv_alias", "-p", "no:cacheprovider",
           "-c", os.devnull, "--rootdir", os.path.join(REF, "tests"), f"--junitxml={xml}",
           *[os.path.join(REF, "tests", f) for f in FILES]]
    out = subprocess.run(cmd, env=_env(), capture_output=True, text=True, timeout=3000)
    cases = {}
    for tc in ET.parse(xml).getroot().iter("testcase"):
        f = tc.get("classname", "").split(".")[-1] + ".py"
        bad = [c.tag for c in tc if c.tag in ("failure", "error", "skipped")]
        cases[(f, tc.get("name"))] = bad[0] if bad else "passed"
    summary = {"passed": sum(v == "passed" for v in cases.values()), "total": len(cases),
               "not_passed": sorted(f"{f}::{n}: {v}" for (f, n), v in cases.items()
                                    if v != "passed")}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ref_conformance.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary))
    for f, names in HOT.items():
        for n in names:
            assert cases.get((f, n)) == "passed", (f, n, out.stdout[-3000:])
    assert summary["passed"] == summary["total"], (summary, out.stdout[-4000:])
