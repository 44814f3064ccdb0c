"""The link-level C++ drop-in (dropin/slicecraft_api.cpp -> libslicecraft_dropin.so):
one caller program written against the reference API (dropin/dropin_cases.cpp)
linked against the drop-in and the product library only, its transcript
compared line by line with the unmodified reference's (tests/golden/dropin_ref.txt,
made by the same program linked against oracle/_ref)."""
import os
import re
import subprocess

import pytest

from conftest import GOLDEN, ROOT

B200 = os.path.join(ROOT, "dropin", "cases_b200")
REF = os.path.join(ROOT, "dropin", "cases_ref")
DROPIN_SO = os.path.join(ROOT, "dropin", "libslicecraft_dropin.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libslicecraft_ref.so")
GOLD = os.path.join(GOLDEN, "dropin_ref.txt")


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.relpath(path, ROOT)} not built (needs the reference headers "
                    "at build time: make dropin)")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference_transcript():
    _need(B200)
    out = subprocess.run([B200, GOLD], capture_output=True, text=True, timeout=900)
    print(out.stdout[-3000:])
    assert out.returncode == 0 and "DROPIN OK" in out.stdout, out.stdout[-3000:] + out.stderr


@pytest.mark.gpu
def test_cpp_dropin_pruned_mode_same_transcript():
    """The implicit context in the exact pruned mode gives the same transcript."""
    _need(B200)
    env = dict(os.environ, SLICECRAFT_B200_MODE="pruned")
    out = subprocess.run([B200, GOLD], capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0 and "DROPIN OK" in out.stdout, out.stdout[-3000:] + out.stderr


def test_cpp_dropin_links_without_the_reference():
    """CPU: the drop-in caller resolves libslicecraft_dropin + libslicecraft_b200
    and nothing built from the reference."""
    _need(B200)
    out = subprocess.run(["ldd", B200], capture_output=True, text=True).stdout
    assert "libslicecraft_dropin.so" in out and "libslicecraft_b200.so" in out
    assert "not found" not in out
    assert "slicecraft_ref" not in out
    out = subprocess.run(["ldd", DROPIN_SO], capture_output=True, text=True).stdout
    assert "slicecraft_ref" not in out and "libslicecraft_b200.so" in out


def _api_symbols(so):
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                        check=True).stdout
    names = [ln.split()[2] for ln in nm.splitlines() if len(ln.split()) == 3 and
             ln.split()[1] == "T"]
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                         check=True).stdout.splitlines()
    return {d for d in dem if d.startswith("slicecraft::") and "b200::" not in d}


def test_cpp_dropin_defines_every_reference_api_symbol():
    """CPU: every function the reference library exports in namespace
    slicecraft (the API of proj/include) is defined by the drop-in."""
    _need(DROPIN_SO)
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    ref = _api_symbols(REF_SO)
    assert len(ref) >= 35
    missing = ref - _api_symbols(DROPIN_SO)
    assert not missing, sorted(missing)


def test_reference_transcript_is_pinned():
    """CPU: the committed golden transcript is what the unmodified reference
    prints (where oracle/_ref and cases_ref exist)."""
    _need(REF)
    out = subprocess.run([REF], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0
    assert out.stdout == open(GOLD).read()
    assert len(re.findall(r"throws", out.stdout)) >= 30  # every error class is exercised
