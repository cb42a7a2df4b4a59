"""The C++ drop-in (include/holoquant/lutham_b200.hpp) against the reference
C++ API itself: tests/cpp/test_lutham_b200.cpp builds host Models with
holoquant::build_model and compares holoquant::compressed_forward /
deserialize / plan_memory (oracle/_ref, the unmodified reference) with the
device head behind the drop-in.  The binary is compiled by
__graft_entry__.build() where /root/reference exists and travels with the
snapshot."""
import os
import subprocess

import pytest

from paper_2512_15742_b200.build import CPP_TEST_BIN, build_cpp_tests


def _binary():
    path = build_cpp_tests()
    if path is None or not os.path.exists(CPP_TEST_BIN):
        pytest.fail("tests/cpp/bin/test_lutham_b200 is missing: run __graft_entry__.build() where "
                    "/root/reference is present")
    return CPP_TEST_BIN


def _run(section):
    r = subprocess.run([_binary(), section], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout, r.stdout
    return r.stdout


def test_cpp_drop_in_planner_and_file_faults():
    out = _run("cpu")
    assert out.count("PASS") == 2


@pytest.mark.gpu
def test_cpp_drop_in_forward_parity_on_device():
    out = _run("gpu")
    assert "FAIL" not in out and out.count("PASS") >= 5
