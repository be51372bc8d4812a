#!/bin/bash
# ASan + UBSan build of the host runtime (s2l_host.cpp) linked with the regular kernel objects,
# then the host-only bookkeeping suites (10,000-step fuzz x3, C1 walks, pressure driver,
# scheduler) through it.  CPU only.  Output: profiles/<round>/asan_ubsan_host.txt
set -e
R=${1:-r02}
cd "$(dirname "$0")/.."
python -m paper_2604_16395_b200.build > /dev/null
mkdir -p /tmp/s2l_asan
g++ -std=c++17 -O1 -g -fsanitize=address,undefined -fno-omit-frame-pointer -fPIC -I include \
    -I paper_2604_16395_b200/csrc -I /usr/local/cuda/include -c paper_2604_16395_b200/csrc/s2l_host.cpp \
    -o /tmp/s2l_asan/s2l_host.o
g++ -shared -fsanitize=address,undefined -o /tmp/s2l_asan/libs2l_asan.so /tmp/s2l_asan/s2l_host.o \
    paper_2604_16395_b200/build/attn_generic.cu.o paper_2604_16395_b200/build/attn_tc.cu.o \
    paper_2604_16395_b200/build/kernels_append.cu.o -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread
S2L_LIB=/tmp/s2l_asan/libs2l_asan.so \
LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)" \
ASAN_OPTIONS=detect_leaks=0:halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
python -m pytest tests/test_host_bookkeeping.py tests/test_pressure.py tests/test_scheduler.py -q -s \
    -p no:cacheprovider 2>&1 | tee profiles/$R/asan_ubsan_host.txt | tail -3
