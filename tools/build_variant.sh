#!/bin/bash
# build a variant library: tools/build_variant.sh <tag> "<nvcc -D flags>"  -> paper_2503_02134_b200/libnb_<tag>.so
tag=$1; shift
NB_NVCC_EXTRA="$*" NB_LIBPATH=$PWD/paper_2503_02134_b200/libnb_$tag.so NB_OBJ_TAG=_$tag \
  python -c "import sys; sys.path.insert(0,'.'); from paper_2503_02134_b200 import _build as b; b.build(force=True)"
