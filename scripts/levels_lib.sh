#!/bin/bash
# run scripts/levels.py against an alternative build of the library: levels_lib.sh <libname> args...
lib=$1; shift
GR_LIB=$lib python scripts/levels.py "$@"
