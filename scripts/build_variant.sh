#!/bin/bash
# build_variant.sh <libname> <nvcc -D flags...>: an alternative build of the
# library for A/B measurements (select it at run time with GR_LIB=<libname>)
lib=$1; shift
GR_NVCC_EXTRA="$*" python -c "
import sys; sys.path.insert(0,'.')
from paper_1501_05387_b200 import _build
_build.build(force=True, lib='paper_1501_05387_b200/$lib')" 2>&1 | grep -i -E ' error|failed'
