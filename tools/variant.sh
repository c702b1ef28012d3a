#!/bin/bash
# A/B kernel experiments: build/var_<name>.so = libmcf.so with als_tc.cu
# patched by sed expressions; run with MCF_LIB=build/var_<name>.so.
#   tools/variant.sh depth1 -e 's/MMA_DEPTH = 2;/MMA_DEPTH = 1;/'
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/var
mkdir -p build/var/$name
src=build/var/$name/als_tc.cu
sed "$@" paper_1108_2580_b200/csrc/als_tc.cu > $src
# MCF_TC_PROFILE=1: compile the phase counters in (tools/tc_phases*.py)
# HSED: a sed expression for als_params.cuh (found next to the patched source first)
if [ -n "$HSED" ]; then sed -e "$HSED" paper_1108_2580_b200/csrc/als_params.cuh > build/var/$name/als_params.cuh
else rm -f build/var/$name/als_params.cuh; fi
cmp -s $src paper_1108_2580_b200/csrc/als_tc.cu && [ -z "$HSED$MCF_TC_PROFILE" ] && { echo "variant $name: patch changed nothing"; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -Xptxas -v --expt-relaxed-constexpr -I paper_1108_2580_b200/csrc -I include \
     ${MCF_TC_PROFILE:+-DMCF_TC_PROFILE} \
     -c -o build/var/$name/als_tc.o $src 2> build/var/$name.ptxas.log
objs=$(ls build/*.o | grep -v '/als_tc.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name.so $objs build/var/$name/als_tc.o -ldl
echo "build/var_$name.so"
