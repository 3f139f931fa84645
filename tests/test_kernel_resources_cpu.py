"""Register / local-memory budget of the hot sm_100a kernels (cuobjdump -res-usage of the built
library): a spill in the QKV epilogue once cost 10% of the TTFT, so the budget is pinned here."""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2512_12977_b200",
                   "libvlcache.so")

# kernel (mangled-name fragment) -> max local-memory bytes per thread (stack)
BUDGET = {
    "gemm_bf16_tcILi6ELi1E": 64,       # QKV GEMM + RoPE epilogue
    "gemm_bf16_tcILi4ELi1E": 0,        # gate/up GEMM + SwiGLU epilogue
    "gemm_bf16_tcILi1ELi1E": 0,        # O / down GEMMs (residual red.add)
    "attn_paged_kernelILi128E": 64,    # paged attention (store chunks rotated in smem)
    "rmsnorm_kernelILb0ELi8E": 0,
}


@pytest.mark.skipif(shutil.which("cuobjdump") is None or not os.path.exists(LIB), reason="no cuobjdump / library")
def test_hot_kernels_do_not_spill():
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    usage = {}
    lines = out.splitlines()
    for i, line in enumerate(lines):
        m = re.search(r"Function (\S+):", line)
        if m and i + 1 < len(lines):
            st = re.search(r"STACK:(\d+)", lines[i + 1])
            rg = re.search(r"REG:(\d+)", lines[i + 1])
            if st and rg:
                usage[m.group(1)] = (int(rg.group(1)), int(st.group(1)))
    for frag, budget in BUDGET.items():
        hits = {k: v for k, v in usage.items() if frag in k}
        assert hits, f"kernel {frag} not found in {LIB}"
        for name, (reg, stack) in hits.items():
            assert stack <= budget, f"{name}: {stack} B of stack (budget {budget}), {reg} registers"
