#!/bin/sh
# ref_tests.sh SRC RANGES OUT -- compile line ranges of one reference test source (read where it
# lies under /root/reference, piped to the compiler, never copied) against include/lkv/ and the
# doctest stand-in, linked to liblkv_b200.so.  `#line` keeps the reference's file:line in messages.
set -e
src=$1; ranges=$2; out=$3
here=$(cd "$(dirname "$0")" && pwd)
{
  for r in $(echo "$ranges" | tr ',' ' '); do
    a=${r%-*}; b=${r#*-}
    echo "#line $a \"$src\""
    sed -n "${a},${b}p" "$src"
  done
} | ${CXX:-g++} -std=c++20 -O1 -w -I"$here/../include" -I"$here/../tests/cpp/doctest_shim" -I"$(dirname "$src")" \
    -x c++ - -o "$out" -L"$here/../paper_2605_06676_b200" -llkv_b200 \
    -Wl,-rpath,'$ORIGIN/../../paper_2605_06676_b200'
