"""SASS-level properties of the built library (CPU: cuobjdump on the
sm_100a cubin): the kernels do what DESIGN.md says they do."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2204_02662_b200", "libpathgcn_b200.so")


def _sass():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe) or not os.path.exists(SO):
        pytest.skip("cuobjdump or the library missing")
    out = subprocess.run([exe, "-sass", SO], capture_output=True, text=True, timeout=300).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


# an instruction whose opcode is a global reduction / atomic (the mbarrier
# SYNCS.ARRIVE.TRANS64.RED of the bulk copy is a shared-memory barrier op)
GLOBAL_ATOMIC = re.compile(r"^\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?(RED|ATOM|ATOMG)\b", re.M)


@pytest.fixture(scope="module")
def sass():
    return _sass()


def _kernels(sass, pat):
    ks = {k: "\n".join(v) for k, v in sass.items() if re.search(pat, k)}
    assert ks, pat
    return ks


def test_grouped_kernel_is_atomic_free_and_stages_records(sass):
    """k_agg_grp (PG_AGG_GROUPED default): no global RED/ATOM; the record
    window arrives by TMA bulk copy (UBLKCP) and is read from shared memory
    (LDS); row gathers are 128-bit (LDG.E.128)."""
    for name, body in _kernels(sass, r"k_agg_grp").items():
        assert not GLOBAL_ATOMIC.search(body), name
        assert "UBLKCP" in body and re.search(r"\bLDS", body), name
        # staged records are read through the shared window, not generic loads
        assert not re.search(r"\bLD\.E", body), name
        assert "LDG.E.128" in body, name
    for name, body in _kernels(sass, r"k_grp_fixup").items():
        assert not GLOBAL_ATOMIC.search(body), name


def test_tensor_core_gemm_uses_tcgen05(sass):
    """k_gemm_abt_tc: tcgen05 MMAs (UTCHMMA for kind::tf32), TMEM loads
    (LDTM), TMA tensor loads (UTMALDG) and bulk copies (UBLKCP)."""
    for name, body in _kernels(sass, r"k_gemm_abt_tc").items():
        for op in ("UTCHMMA", "LDTM", "UTMALDG", "UBLKCP"):
            assert op in body, (name, op)


def test_register_tiled_gemm_is_unfused_and_async_staged(sass):
    """k_gemm3 (the default bit-exact GEMM): products as FFMA2 with a -0
    addend plus FADD2 (no fused multiply-add into the chain), A / B tiles by
    cp.async (LDGSTS) into shared memory, read back as LDS.128."""
    for name, body in _kernels(sass, r"k_gemm3").items():
        assert re.search(r"\bFFMA2\b", body) and re.search(r"\bFADD2\b", body), name
        assert "LDGSTS" in body and "LDS.128" in body, name
        assert not re.search(r"\bFFMA\b", body), name  # no scalar fused chain step


def test_default_spmm_gathers_are_128_bit(sass):
    """k_agg_vec4 (default instantiation) and the whole-row k_agg_row gather
    rows with 128-bit loads and keep the multiply and the add separate."""
    for pat in (r"k_agg_vec4ILi32ELi8ELb0ELi0ELb0ELi256E", r"k_agg_rowILi5ELi2E"):
        for name, body in _kernels(sass, pat).items():
            assert "LDG.E.128" in body, name
            assert re.search(r"\bFADD2\b", body), name
            assert not GLOBAL_ATOMIC.search(body), name


def test_wide_spmm_gathers_are_256_bit(sass):
    """k_agg_vec8 (the wide-row default from 2^21 edges per call): every
    row gather one 256-bit load per lane and edge (LDG.E.ENL2.256), the unfused
    FFMA2 + FADD2 chain step, no spills, no global atomics."""
    for name, body in _kernels(sass, r"k_agg_vec8ILi4E").items():
        # U = 4 gathers in the batch loop + 4 in the remainder batch (the
        # two LDG.E.128 left are the accumulate-mode output loads)
        assert len(re.findall(r"LDG\.E\.ENL2\.256", body)) >= 8, name
        assert re.search(r"\bFFMA2\b", body) and re.search(r"\bFADD2\b", body), name
        assert not re.search(r"\b(STL|LDL)\b", body), name
        assert not GLOBAL_ATOMIC.search(body), name


def test_f64_wide_gathers_are_256_bit_and_unfused(sass):
    """k_agg_f64v (aggregate_pull<double>, rows > 32 doubles): 256-bit row
    gathers; every multiply and add separately rounded (DMUL + DADD, no DFMA
    — the reference's default-flag x86-64 build does not contract)."""
    for name, body in _kernels(sass, r"k_agg_f64v?ILi").items():
        assert re.search(r"\bDMUL\b", body) and re.search(r"\bDADD\b", body), name
        assert not re.search(r"\bDFMA\b", body), name
        assert not re.search(r"\b(STL|LDL)\b", body), name
    for name, body in _kernels(sass, r"k_agg_f64vILi4E").items():
        assert len(re.findall(r"LDG\.E\.ENL2\.256", body)) >= 8, name
