#!/bin/bash
# Build libmgk variants for A/B timing on the GPU box:
#   tools/build_variants.sh NAME "-DMGK_PANEL_SLOTS=8 -DMGK_PANEL_PIPELINE=0" ...
# capi.cu, pcg_warp.cu and both panel-solver objects get the extra defines; the other translation units come
# from the default build.
set -e
cd "$(dirname "$0")/../paper_1910_06310_b200"
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Icsrc -I../include"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  mkdir -p build/$name
  $NVCC $FL $defs -c csrc/capi.cu -o build/$name/capi.o &
  $NVCC $FL $defs -c csrc/pcg_warp.cu -o build/$name/pcg_warp.o &
  $NVCC $FL -DMGK_PANEL_THREADS=256 -DMGK_PANEL_NS=p256 $defs -c csrc/pcg_panel.cu -o build/$name/pcg_panel_256.o &
  $NVCC $FL -DMGK_PANEL_THREADS=512 -DMGK_PANEL_NS=p512 $defs -c csrc/pcg_panel.cu -o build/$name/pcg_panel_512.o &
  wait
  objs="build/$name/capi.o build/$name/pcg_warp.o build/$name/pcg_panel_256.o build/$name/pcg_panel_512.o"
  for f in tiles pcg_block pbr bench_support gram_post ingest order; do objs="$objs build/$f.o"; done
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o libmgk_$name.so $objs -lcudart
  echo built libmgk_$name.so
done
