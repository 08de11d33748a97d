"""C-ABI checks that need no GPU: the library loads, exports every function include/tag.h declares,
the host-only selector is bit-exact against the oracle, and argument validation fails cleanly."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tagmod():
    from paper_2302_06126_b200 import tag
    return tag


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "tag.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tag_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(tagmod):
    declared = _declared_functions()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(tagmod._lib, name), name
    assert set(declared) == set(tagmod.EXPORTS)


def test_exports_match_nm(tagmod):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", tagmod.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (tag_[a-z0-9_]+)", out))
    assert exported == set(_declared_functions())
    # the library is built for sm_100a only
    sass = subprocess.run(["cuobjdump", "--list-elf", tagmod.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass


def test_version_and_status_strings(tagmod):
    assert "sm_100a" in tagmod.version()
    assert tagmod._lib.tag_status_string(tagmod.ERR_INVALID_ARG) == b"TAG_ERR_INVALID_ARG"
    assert tagmod._lib.tag_status_string(99) == b"TAG_ERR_UNKNOWN"


def test_select_matches_oracle_appendix_a(tagmod, oracle_mod):
    import json
    S = oracle_mod.selector
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "appendix_a_decisions.json")))
    for c in cases["cases"]:
        lay = dict(M=c["M"], N=c["N"], B=c["B"], factor_dtype="f32" if c["e_w"] == 4 else "bf16",
                   grad_dtype="f32" if c["e_g"] == 4 else "bf16")
        got = tagmod.select([lay], c["n"], c["tau"], c["F"], c["rule"])[0]
        want = S.select(dict(M=c["M"], N=c["N"], B=c["B"], e_w=c["e_w"], e_g=c["e_g"]),
                        dict(n=c["n"], tau=c["tau"], F=c["F"], rule=c["rule"]))
        assert got == want, c


def test_select_random_bit_exact(tagmod, oracle_mod):
    S = oracle_mod.selector
    rs = np.random.default_rng(11)
    for _ in range(400):
        L = int(rs.integers(1, 6))
        lays = [dict(M=int(rs.integers(1, 60000)), N=int(rs.integers(1, 60000)),
                     B=int(rs.integers(1, 4096)), e_w=int(rs.choice([2, 4])),
                     e_g=int(rs.choice([2, 4]))) for _ in range(L)]
        n = int(rs.integers(1, 65))
        tau = int(rs.integers(1, 2 * 10 ** 12))
        F = int(rs.choice([0, int(rs.integers(1, 4 * 10 ** 15))]))
        rule = int(rs.integers(0, 3))
        dt = {2: "bf16", 4: "f32"}
        got = tagmod.select([dict(M=l["M"], N=l["N"], B=l["B"], factor_dtype=dt[l["e_w"]],
                                  grad_dtype=dt[l["e_g"]]) for l in lays], n, tau, F, rule)
        want = [S.select(l, dict(n=n, tau=tau, F=F, rule=rule)) for l in lays]
        assert got == want


def test_select_knife_edges(tagmod, oracle_mod):
    """Exact ties and one-unit neighbours: the library must agree with exact arithmetic."""
    S = oracle_mod.selector
    # tie (S:506 -> AllReduce): n^2 S = 2(n-1) G at M = N = 16, B = 4, bf16/bf16, n = 2
    assert tagmod.select([dict(M=16, N=16, B=4, factor_dtype="bf16", grad_dtype="bf16")], 2,
                         10 ** 9, 0)[0] == tagmod.SYNC_ALLREDUCE
    assert tagmod.select([dict(M=16, N=16, B=3, factor_dtype="bf16", grad_dtype="bf16")], 2,
                         10 ** 9, 0)[0] == tagmod.SYNC_SFB
    # Transformer FFN at n = 4 with the compute term: 6.96 us vs 6.99 us
    lay = dict(M=512, N=2048, B=256)
    for F in (1421400000000000, 10 ** 15, 2 * 10 ** 15):
        for tau in (9 * 10 ** 11, 8 * 10 ** 11, 77 * 10 ** 10):
            got = tagmod.select([dict(lay, factor_dtype="bf16", grad_dtype="f32")], 4, tau, F)[0]
            assert got == S.select(dict(lay, e_w=2, e_g=4), dict(n=4, tau=tau, F=F))


def test_select_n1_and_errors(tagmod):
    assert tagmod.select([dict(M=4, N=4, B=1)], 1) == [tagmod.SYNC_NONE]
    with pytest.raises(tagmod.TagError) as e:
        tagmod.select([dict(M=0, N=4, B=1)], 2)
    assert e.value.status == tagmod.ERR_INVALID_ARG
    with pytest.raises(tagmod.TagError):
        tagmod.select([dict(M=4, N=4, B=1)], 2, link_bytes_per_s=0)
    with pytest.raises(tagmod.TagError):
        tagmod.select([dict(M=4, N=4, B=1)], 2, rule=7)
    assert tagmod.select([], 2) == []
    # overflow is reported, never wrapped
    with pytest.raises(tagmod.TagError) as e:
        tagmod.select([dict(M=2 ** 40, N=2 ** 40, B=2 ** 30)], 64, 2 ** 63, 2 ** 63)
    assert e.value.status == tagmod.ERR_UNSUPPORTED


def test_no_gpu_means_loud_failure(tagmod):
    """Without a CUDA device the compute path must fail, never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tagmod.TagError) as e:
        tagmod.Comm(1, 0, 0)
    assert e.value.status in (tagmod.ERR_CUDA, tagmod.ERR_INVALID_ARG)


def test_select_profiled_bit_exact(tagmod, oracle_mod):
    S = oracle_mod.selector
    rs = np.random.default_rng(31)
    dt = {2: "bf16", 4: "f32"}
    for _ in range(300):
        npts = int(rs.integers(2, 8))
        def curve():
            b = np.cumsum(rs.integers(1, 10 ** 8, npts)).tolist()
            t = rs.integers(1000, 10 ** 7, npts).tolist()
            return list(zip(b, t))
        g, a = curve(), curve()
        n = int(rs.integers(1, 17))
        F = int(rs.choice([0, int(rs.integers(10 ** 12, 3 * 10 ** 15))]))
        lays = [dict(M=int(rs.integers(1, 30000)), N=int(rs.integers(1, 30000)),
                     B=int(rs.integers(1, 2048)), e_w=int(rs.choice([2, 4])),
                     e_g=int(rs.choice([2, 4]))) for _ in range(4)]
        got = tagmod.select_profiled([dict(M=l["M"], N=l["N"], B=l["B"], factor_dtype=dt[l["e_w"]],
                                           grad_dtype=dt[l["e_g"]]) for l in lays], n, g, a, F)
        want = [S.select_profiled(l, n, g, a, F) for l in lays]
        assert got == want


def test_select_profiled_measured_times_bit_exact(tagmod, oracle_mod):
    """f-4: measured per-layer op times (recon at K = nB, local gradient at K = B) in the profiled
    selector, library == oracle, with and without the PS curve."""
    S = oracle_mod.selector
    rs = np.random.default_rng(37)
    dt = {2: "bf16", 4: "f32"}
    seen = set()
    for _ in range(300):
        def curve():
            b = np.cumsum(rs.integers(1, 10 ** 8, int(rs.integers(2, 6)))).tolist()
            return list(zip(b, rs.integers(1000, 10 ** 7, len(b)).tolist()))
        g, a, ps = curve(), curve(), (curve() if rs.integers(0, 2) else None)
        n = int(rs.integers(1, 9))
        lays = [dict(M=int(rs.integers(1, 30000)), N=int(rs.integers(1, 30000)),
                     B=int(rs.integers(1, 2048)), e_w=int(rs.choice([2, 4])),
                     e_g=int(rs.choice([2, 4]))) for _ in range(4)]
        rec = [int(rs.integers(0, 10 ** 7)) for _ in lays]
        loc = [int(rs.integers(0, 10 ** 6)) for _ in lays]
        got = tagmod.select_profiled([dict(M=l["M"], N=l["N"], B=l["B"], factor_dtype=dt[l["e_w"]],
                                           grad_dtype=dt[l["e_g"]]) for l in lays], n, g, a, 10 ** 15,
                                     ps, recon_ns=rec, local_ns=loc)
        want = [S.select_profiled(l, n, g, a, 10 ** 15, ps, recon_ns=r, local_ns=o)
                for l, r, o in zip(lays, rec, loc)]
        assert got == want
        seen.update(got)
    assert {tagmod.SYNC_ALLREDUCE, tagmod.SYNC_SFB, tagmod.SYNC_NONE} <= seen
    with pytest.raises(tagmod.TagError):
        tagmod.select_profiled([dict(M=4, N=4, B=1)], 2, [(1, 1), (2, 2)], [(1, 1), (2, 2)],
                               recon_ns=[1 << 41], local_ns=[0])


def test_select_profiled_errors(tagmod):
    with pytest.raises(tagmod.TagError):
        tagmod.select_profiled([dict(M=4, N=4, B=1)], 2, [(1, 1)], [(1, 1), (2, 2)])   # 1 point
    with pytest.raises(tagmod.TagError):
        tagmod.select_profiled([dict(M=4, N=4, B=1)], 2, [(2, 1), (1, 2)], [(1, 1), (2, 2)])
    assert tagmod.select_profiled([dict(M=4, N=4, B=1)], 1, [(1, 1), (2, 2)],
                                  [(1, 1), (2, 2)]) == [tagmod.SYNC_NONE]


def test_select_profiled_with_ps_bit_exact(tagmod, oracle_mod):
    """Three-way profiled decision (AllReduce / SFB / Replicate-with-PS) equals the oracle's."""
    S = oracle_mod.selector
    rs = np.random.default_rng(33)
    dt = {2: "bf16", 4: "f32"}
    seen = set()
    for _ in range(400):
        def curve():
            b = np.cumsum(rs.integers(1, 10 ** 8, int(rs.integers(2, 6)))).tolist()
            t = rs.integers(1000, 10 ** 7, len(b)).tolist()
            return list(zip(b, t))
        g, a, ps = curve(), curve(), curve()
        n = int(rs.integers(2, 9))
        lays = [dict(M=int(rs.integers(1, 30000)), N=int(rs.integers(1, 30000)),
                     B=int(rs.integers(1, 2048)), e_w=int(rs.choice([2, 4])),
                     e_g=int(rs.choice([2, 4]))) for _ in range(4)]
        got = tagmod.select_profiled([dict(M=l["M"], N=l["N"], B=l["B"], factor_dtype=dt[l["e_w"]],
                                           grad_dtype=dt[l["e_g"]]) for l in lays], n, g, a, 0, ps)
        want = [S.select_profiled(l, n, g, a, 0, ps) for l in lays]
        assert got == want
        seen.update(got)
    assert seen == {tagmod.SYNC_ALLREDUCE, tagmod.SYNC_SFB, tagmod.SYNC_PS}
    with pytest.raises(tagmod.TagError):
        tagmod.select_profiled([dict(M=4, N=4, B=1)], 2, [(1, 1), (2, 2)], [(1, 1), (2, 2)], 0,
                               [(2, 1), (1, 2)])                       # PS bytes not increasing


def _build_c_example(tmp_path):
    import subprocess
    exe = str(tmp_path / "c_abi_example")
    lib_dir = os.path.join(ROOT, "paper_2302_06126_b200")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_abi_example.c"),
                    "-o", exe, "-L", lib_dir, "-ltag", f"-Wl,-rpath,{lib_dir}",
                    "-L", "/usr/local/cuda/lib64", "-lcudart"], check=True)
    return exe


def test_c_program_uses_the_abi(tmp_path, tagmod):
    """include/tag.h is plain C11 and libtag links into a C program; its host-only calls
    (selector, ILP, argument validation) run without a GPU."""
    import subprocess
    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe, "--host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fc6 -> SFB" in r.stdout and "objective = -9.700e-04" in r.stdout


@pytest.mark.gpu
def test_c_program_sync_on_gpu(tmp_path, tagmod):
    """The same C program runs one SFB sync on GPU 0 and checks every element exactly."""
    import subprocess
    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
