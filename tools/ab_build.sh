#!/bin/bash
# A/B builds of the library: tools/ab_build.sh OUT.so [extra nvcc flags...]
# compiles rbf_gcb.cu with the extra flags (e.g. -DRBF_OV_SLEEP_NS=100) and
# links it with the other sources (compiled once into /tmp/ab_objs).
set -e
out=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2004_04817_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -Xcompiler -fvisibility=hidden"
mkdir -p /tmp/ab_objs
for s in rbf_capi rbf_eval rbf_chol; do
  [ /tmp/ab_objs/$s.o -nt $C/$s.cu ] || nvcc $F -c $C/$s.cu -o /tmp/ab_objs/$s.o
done
[ /tmp/ab_objs/rbf_meshio.o -nt $C/rbf_meshio.cpp ] || g++ -O3 -std=c++17 -fPIC -fvisibility=hidden -pthread -I /usr/local/cuda/include -c $C/rbf_meshio.cpp -o /tmp/ab_objs/rbf_meshio.o
nvcc $F "$@" -c $C/rbf_gcb.cu -o /tmp/ab_objs/gcb_v.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" /tmp/ab_objs/rbf_capi.o /tmp/ab_objs/rbf_eval.o /tmp/ab_objs/rbf_chol.o /tmp/ab_objs/gcb_v.o /tmp/ab_objs/rbf_meshio.o -lcudart_static -lrt -lpthread -ldl
