#!/bin/bash
# Rebuild only the named objects (e.g. `tools/quick_build.sh kernels_4step_f32 host`) and relink the
# library: the Makefile's header dependencies rebuild every TU (13 minutes) when any header changes.
# EXTRA="-D..." is passed to nvcc; the named objects are always recompiled.
set -e
cd "$(dirname "$0")/../paper_2108_03948_b200/csrc"
objs=()
for n in "$@"; do
    objs+=("../build/$n.o")
    rm -f "../build/$n.o"
done
if [ ${#objs[@]} -gt 0 ]; then
    make -s -j8 "${objs[@]}" OBJDIR=../build EXTRA="$EXTRA" 2>&1 | grep -v "Registers are spilled" || true
fi
mkdir -p ../lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libspectralkit_b200.so ../build/*.o
echo linked
