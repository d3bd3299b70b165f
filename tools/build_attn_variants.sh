#!/bin/bash
# A/B builds of the decode attention alternatives (k_attn_decode.cu build-time switches): one
# full libquota_b200.so per variant under paper_2604_17320_b200/_build_var/<name>/, selected at
# run time with QT_LIB_PATH (the Python binding's override).
set -e
cd "$(dirname "$0")/.."
B=paper_2604_17320_b200/_build
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
make -C paper_2604_17320_b200/csrc -j8 > /dev/null
OTHERS=$(ls $B/*.o | grep -v k_attn_decode.o)
for v in "pw1fq:-DQT_AD_KERNEL=1 -DQT_AD_CTAS=1 -DQT_AD_FUSEQ=1" "pw1:-DQT_AD_KERNEL=1 -DQT_AD_CTAS=1 -DQT_AD_FUSEQ=0" \
         "pw2:-DQT_AD_KERNEL=1 -DQT_AD_CTAS=2 -DQT_AD_FUSEQ=0" "tp2:-DQT_AD_KERNEL=2 -DQT_AD_CTAS=2 -DQT_AD_FUSEQ=0" \
         "tp1:-DQT_AD_KERNEL=2 -DQT_AD_CTAS=1 -DQT_AD_FUSEQ=0"; do
  name=${v%%:*}; defs=${v#*:}
  out=paper_2604_17320_b200/_build_var/$name; mkdir -p $out
  /usr/local/cuda/bin/nvcc $FLAGS $defs -c paper_2604_17320_b200/csrc/k_attn_decode.cu -o $out/k_attn_decode.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared $OTHERS $out/k_attn_decode.o -o $out/libquota_b200.so -lcudart -lcublas -Xlinker -rpath,/usr/local/cuda/lib64
  echo built $name
done
