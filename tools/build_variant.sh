#!/bin/bash
# build a variant of libosam.so into ab/<name>.so with extra nvcc flags (A/B timing: tools/ab_bench.sh)
#   bash tools/build_variant.sh NAME [-DFLAG ...]
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p ab
C=paper_2511_20687_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" -o ab/$name.so \
  $C/osam_api.cu $C/kernels_fom.cu $C/kernels_xfer_rom.cu $C/kernels_rom_tc.cu $C/kernels_replay.cu
