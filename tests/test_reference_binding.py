"""The reference-side binding include/bdsm_gpu_reference.hpp:
compiled against the reference's own headers (/root/reference/proj/include),
linked with the unmodified reference library, and driven by the reference's
own fixtures (tests/support/fig1.hpp, random_instances.hpp) with its
match_batch (coalesce off) as the expected result (oracle/ref_binding_check.cpp).

CPU: the header compiles against the reference and, without a GPU, the
binding maps the engine's BDSM_CUDA_ERROR to std::runtime_error.
GPU: every count equals the reference's, including several queries per engine,
and BatchError carries the reference's own failure reasons.
"""
import json
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
CHECK = os.path.join(REPO, "oracle", "_ref", "ref_binding_check")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference sources absent (GPU box)")
def test_binding_header_compiles_against_reference(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "bdsm_gpu_reference.hpp"\nint main() { return 0; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror", f"-I{REF_INC}",
                        f"-I{os.path.join(REPO, 'include')}", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _run():
    if not os.path.exists(CHECK):
        pytest.skip("oracle/_ref/ref_binding_check not built (make -C oracle ref)")
    r = subprocess.run([CHECK], capture_output=True, text=True, timeout=600)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return r.returncode, (json.loads(line[-1]) if line else {}), r.stderr


def test_binding_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc, out, err = _run()
    assert rc == 3 and out.get("no_gpu") is True, (rc, out, err)


@pytest.mark.gpu
def test_binding_equals_reference_match_batch():
    rc, out, err = _run()
    assert rc == 0, (out, err[-2000:])
    assert out["mismatches"] == 0 and out["checks"] > 100 and out["random_streams"] == 40
