#!/bin/bash
# Build libmgk variants of the panel solver for A/B timing on the GPU box:
#   tools/build_variants.sh NAME "-DMGK_PANEL_SLOTS=8 -DMGK_PANEL_PIPELINE=0" ...
# Objects of the other translation units come from the default build.
set -e
cd "$(dirname "$0")/../paper_1910_06310_b200"
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Icsrc -I../include"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  mkdir -p build/$name
  for f in capi pcg_panel; do $NVCC $FL $defs -c csrc/$f.cu -o build/$name/$f.o & done
  wait
  objs="build/$name/capi.o build/$name/pcg_panel.o"
  for f in tiles pcg_warp pcg_block pbr bench_support gram_post ingest; do objs="$objs build/$f.o"; done
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o libmgk_$name.so $objs -lcudart
  echo built libmgk_$name.so
done
