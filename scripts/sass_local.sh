#!/bin/bash
# usage: scripts/sass_local.sh <file.cu> <function-substring>  -> local-memory ops per source line
set -e
cd /root/repo/paper_2106_04487_b200
rm -rf /tmp/sassq && mkdir -p /tmp/sassq
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --expt-relaxed-constexpr -Xcompiler -fPIC -Icsrc -I../include $3 -c "$1" -o /tmp/sassq/k.o -Xptxas -v 2>&1 | grep -A3 "Compiling entry.*$2" | grep -E "stack|Used" || true
cd /tmp/sassq && cuobjdump -xelf all k.o > /dev/null && nvdisasm -g -c *.cubin > k.sass
python3 /root/repo/scripts/ldl.py /tmp/sassq/k.sass "$2"
