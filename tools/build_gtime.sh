#!/bin/bash
# Diagnostics build: libpod_gtime.so with the POD_EXP_GTIME globaltimer stamps (tools/gap_probe.py,
# tools/fused_probe.py; select it with POD_LIB_PATH=paper_2111_05188_b200/libpod_gtime.so)
cd "$(dirname "$0")/.." && python - <<'PY'
import subprocess, sys
sys.path.insert(0, '.')
from paper_2111_05188_b200 import _build
cmd = _build.nvcc_cmd('paper_2111_05188_b200/libpod_gtime.so')
r = subprocess.run(cmd[:1] + ['-DPOD_EXP_GTIME'] + cmd[1:], capture_output=True, text=True)
sys.stderr.write(r.stderr[-2000:] if r.returncode else '')
sys.exit(r.returncode)
PY
