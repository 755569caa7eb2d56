"""SURVEY §4.3 item 6 (host side): the oracle's pins re-run against an
AddressSanitizer + UndefinedBehaviorSanitizer build of oracle/ndgi_oracle.c
(gcc -fsanitize=address,undefined -fno-sanitize-recover=all), in a subprocess
with the ASan runtime preloaded -- any out-of-bounds access, use after free or
undefined behaviour (signed overflow, bad shift, misaligned load) in the
oracle aborts the run.  compute-sanitizer is closed on the GPU pool; the
device side has the self-checking build instead (test_gpu_selfcheck.py)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gcc_file(name):
    return subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()


@pytest.mark.timeout(600)
def test_oracle_pins_under_asan_ubsan(tmp_path):
    asan = _gcc_file("libasan.so")
    if not os.path.isabs(asan) or not os.path.exists(asan):
        pytest.skip("libasan not available")
    lib = str(tmp_path / "liboracle_san.so")
    subprocess.check_call(
        ["gcc", "-O1", "-g", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fPIC", "-shared",
         "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer",
         "-o", lib, os.path.join(ROOT, "oracle", "ndgi_oracle.c"), "-lm", "-lpthread"])
    env = dict(os.environ, ORACLE_LIB=lib, LD_PRELOAD=asan,
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    tests = ["tests/test_oracle_bc7.py", "tests/test_oracle_bcn.py", "tests/test_oracle_sampling.py",
             "tests/test_oracle_mlp.py", "tests/test_oracle_pipeline.py", "tests/test_oracle_shading.py",
             "tests/test_oracle_bc7_encode.py", "tests/test_oracle_train.py", "tests/test_oracle_export.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "ERROR: AddressSanitizer" not in tail and "runtime error" not in tail, tail
