#!/bin/bash
# Build a library variant with extra nvcc defines into build_var/:
#   tools/build_variant.sh name -DFOO -DBAR=2
name=$1; shift
flags=$(python -c "import sys; sys.path.insert(0,'.'); from paper_1904_02833_b200 import _native as n; print(' '.join(n.NVCC_FLAGS))")
mkdir -p build_var
nvcc $flags "$@" -o build_var/$name.so paper_1904_02833_b200/csrc/ss_api.cu
