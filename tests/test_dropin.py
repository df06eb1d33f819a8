"""The reference's own unit tests (test_retriever.cpp, test_streamer.cpp from
/root/reference/proj/tests, compiled unchanged with the doctest shim in
oracle/doctest) linked against the B200 C++ drop-in
(paper_2603_08453_b200/cpp/tierkv_dropin.cpp: tierkv::retrieve / StreamState
over the C ABI) instead of the reference's retriever.o / streamer.o.

The binaries are built in this container by `make -C oracle droptests`
(__graft_entry__.build() does it when /root/reference is present) and travel
to the GPU box in oracle/_ref/.  The same sources linked against the reference
library (`make -C oracle reftests`) validate the shim on the CPU.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _run(binary, timeout):
    path = os.path.join(REF, binary)
    if not os.path.exists(path):
        pytest.skip(f"{binary} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=REF)
    summary = [l for l in r.stdout.splitlines() if "[doctest-shim]" in l]
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert summary and "0 failed | assertions" in summary[-1], summary
    return summary[-1]


@pytest.mark.parametrize("name", ["test_retriever", "test_streamer", "test_kernels", "test_index"])
def test_reference_tests_pass_against_reference_with_shim(name):
    _run(f"ref_{name}", 600)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_retriever", "test_streamer"])
def test_reference_tests_pass_against_b200_dropin(name):
    print(_run(f"b200_{name}", 900))


@pytest.mark.gpu
def test_reference_acceptance_suite_passes_against_b200_dropin():
    """acceptance.cpp's 12 criteria (UB soundness fuzz, degeneracy, recall
    monotonicity, streaming stability, graft caps, byte-identical reruns...)
    with every retrieve() / StreamState call on the B200 drop-in."""
    path = os.path.join(REF, "b200_acceptance")
    if not os.path.exists(path):
        pytest.skip("b200_acceptance not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900, cwd=REF)
    assert r.returncode == 0, r.stdout[-4000:]
    assert "0 of 12 criteria failed" in r.stdout, r.stdout[-4000:]
