#!/bin/bash
# build_variant.sh NAME "<extra nvcc -D flags>" [file.cu ...]: libcamg variant in paper_1912_09056_b200/ab/libcamg_NAME.so
# (the named sources recompiled with the flags -- default sell.cu -- linked with the default objects); use with CAMG_LIB
set -e
name=$1; flags=$2; shift 2 || true
files=${@:-sell.cu}
cd "$(dirname "$0")/../paper_1912_09056_b200/csrc"
mkdir -p ../ab/build_$name
objs=""
for f in sell.cu csr.cu spgemm.cu hierarchy.cu krylov.cu aggregate.cu generator.cu pointsolve.cu hostqr.cu tentqr.cu; do
  if [[ " $files " == *" $f "* ]]; then
    /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 \
      --expt-relaxed-constexpr -Xptxas -v $flags -c $f -o ../ab/build_$name/${f%.cu}.o 2> ../ab/build_$name/${f%.cu}.ptxas.log
    objs="$objs ../ab/build_$name/${f%.cu}.o"
  else
    objs="$objs build/${f%.cu}.o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../ab/libcamg_$name.so $objs -lcudart -ldl
echo built ab/libcamg_$name.so
