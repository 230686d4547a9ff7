#!/bin/bash
# Build library variants for A/B timing: ab_build.sh NAME "-DFLAG ..." -> abtest/libNAME.so
set -e
cd "$(dirname "$0")/.."
HS_NVCC_FLAGS="$2" python -c "from paper_2604_16864_b200 import build; build.build(force=True)" > /dev/null
cp paper_2604_16864_b200/lib/libhierasparse_b200.so abtest/lib$1.so
