#!/bin/bash
# A/B builds of decode attention settings (k_attn_decode.cu build-time defines): one
# full libquota_b200.so per variant under paper_2604_17320_b200/_build_var/<name>/, selected at
# run time with QT_LIB_PATH (the Python binding's override).
set -e
cd "$(dirname "$0")/.."
B=paper_2604_17320_b200/_build
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
make -C paper_2604_17320_b200/csrc -j8 > /dev/null
SRC=${VARIANT_SRC:-k_attn_decode}   # the csrc/<SRC>.cu file the variants rebuild
OTHERS=$(ls $B/*.o | grep -v "/$SRC.o")
# VARIANTS: ';'-separated name:defines list
IFS=';' read -ra VL <<< "${VARIANTS:-base:}"
for v in "${VL[@]}"; do
  name=${v%%:*}; defs=${v#*:}
  out=paper_2604_17320_b200/_build_var/$name; mkdir -p $out
  /usr/local/cuda/bin/nvcc $FLAGS $defs -c paper_2604_17320_b200/csrc/$SRC.cu -o $out/$SRC.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared $OTHERS $out/$SRC.o -o $out/libquota_b200.so -lcudart -lcublas -Xlinker -rpath,/usr/local/cuda/lib64
  echo built $name
done
