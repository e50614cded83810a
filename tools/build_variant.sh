#!/bin/bash
# build_variant.sh NAME "EXTRA NVCC FLAGS" — an alternative build of the
# library under paper_2006_06281_b200/variants/NAME/ (A/B experiments; run
# with FCPD_LIB=.../libfcpd_b200.so)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
D=/tmp/fcpd_variant_$1
rm -rf $D && mkdir -p $D && cp -r $R/paper_2006_06281_b200/csrc $R/paper_2006_06281_b200/Makefile $D/
mkdir -p $D/cli && cp $R/paper_2006_06281_b200/cli/* $D/cli/
sed -i "s|^NVFLAGS := \$(ARCH)|NVFLAGS := \$(ARCH) $2|; s|^ROOT := .*|ROOT := $R|" $D/Makefile
make -s -j8 -C $D $D/lib/libfcpd_b200.so
mkdir -p $R/paper_2006_06281_b200/variants/$1
cp $D/lib/libfcpd_b200.so $R/paper_2006_06281_b200/variants/$1/
grep -A2 "estep_row_kernelILi2" $D/build/estep.ptxas.txt | grep -E "spill|registers"
