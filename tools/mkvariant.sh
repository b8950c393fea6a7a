#!/bin/bash
# Build a variant of libinfllm_b200.so with one source edit, for tools/lib_ab.py:
#   tools/mkvariant.sh NAME FILE 'sed-expression'   -> tmp_libs/libNAME.so
set -e
name=$1; file=$2; expr=$3
root=/tmp/var_$name
rm -rf $root && mkdir -p $root/pkg
cp -r include $root/
cp -r paper_2402_04617_b200/csrc paper_2402_04617_b200/Makefile $root/pkg/
sed -i "$expr" $root/pkg/csrc/$file
if diff -q paper_2402_04617_b200/csrc/$file $root/pkg/csrc/$file > /dev/null; then echo "no change"; exit 1; fi
make -s -C $root/pkg -j8 libinfllm_b200.so
mkdir -p tmp_libs && cp $root/pkg/libinfllm_b200.so tmp_libs/lib$name.so
echo built tmp_libs/lib$name.so
