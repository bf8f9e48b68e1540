#!/bin/bash
# usage: mkvariant.sh NAME [git-rev|-|DIR] [nvcc -D flags...]   (debug aid: builds a variant package
# from the working tree (-), a git revision, or a patched copy DIR made for the *_trace_patch.py scripts)
set -e
name=$1; rev=$2; shift 2
d=/root/repo/scripts/debug/variants/$name/paper_2003_02978_b200
mkdir -p $d
if [ "$rev" = "-" ]; then src=/root/repo; elif [ -d "$rev" ]; then src=$rev; else src=/tmp/mkv_$name; mkdir -p $src; git -C /root/repo archive $rev paper_2003_02978_b200 include | tar -x -C $src; fi
cp $src/paper_2003_02978_b200/*.py $d/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static "$@" -o $d/libsmf.so $src/paper_2003_02978_b200/csrc/smf.cu
touch $d/libsmf.so
