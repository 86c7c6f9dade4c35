#!/bin/bash
# tools/mkvariant.sh NAME "nvcc extra flags": build libcmf_b200.so with the flags into tools/ab/NAME.so
set -e
mkdir -p tools/ab
CMF_NVCC_EXTRA="$2" python -m paper_1808_03843_b200._build > /dev/null
cp paper_1808_03843_b200/libcmf_b200.so tools/ab/$1.so
echo "built tools/ab/$1.so ($2)"
