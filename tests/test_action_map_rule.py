"""The fused rollout kernel decides the action map floor(|u| h_max + 1/2) (R#6, a float64 expression) in
float32 when a margin proves it equal to the float64 result, and redoes it in float64 otherwise
(csrc/actor_kernel.cuh, the head).  This checks that rule exhaustively on the host, over every float32
|u| in [0, 1] for h_max = 100 (and strided for other h_max <= 128): whenever the float32 path is taken
(the fractional part of fl32(|u| h_max + 1/2) lies in [2^-15, 1 - 2^-15]) it equals the float64 floor."""
import os
import subprocess

import pytest

SRC = r'''
#include <cmath>
#include <cstdio>
#include <cstring>
int main() {
    const int hs[] = {100, 1, 3, 7, 64, 127, 128};
    long long bad = 0, unsure = 0, n = 0;
    for (int hi = 0; hi < 7; ++hi) {
        const int h = hs[hi];
        const float hf = static_cast<float>(h);
        const unsigned step = h == 100 ? 1u : 61u;
        for (unsigned b = 0; b <= 0x3f800000u; b += step) {
            float u;
            std::memcpy(&u, &b, 4);
            const float r = std::fmaf(u, hf, 0.5f);   // the kernel's fmaf(fabsf(u), hmax_f, 0.5f)
            const float fl = std::floor(r);
            const float d = r - fl;
            ++n;
            if (d < 3.0517578125e-05f || d > 0.999969482421875f) { ++unsure; continue; }
            const double ref = std::floor(static_cast<double>(u) * static_cast<double>(h) + 0.5);
            if (static_cast<int>(fl) != static_cast<int>(ref)) {
                if (bad < 5) std::printf("mismatch h=%d bits=%08x\n", h, b);
                ++bad;
            }
        }
    }
    std::printf("checked %lld unsure %lld bad %lld\n", n, unsure, bad);
    return bad != 0;
}
'''


def test_float32_action_map_rule(tmp_path):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        pytest.skip("nvcc missing")
    src = tmp_path / "rule.cu"
    src.write_text(SRC)
    exe = tmp_path / "rule"
    subprocess.run([nvcc, "-O2", "-o", str(exe), str(src)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " bad 0" in r.stdout
