#!/bin/bash
# Snapshot the current in-tree build as build_ab/NAME.so (for tools/ab_build.sh).
set -e
make -C paper_2511_15022_b200/csrc -j8 >/dev/null
mkdir -p build_ab
cp paper_2511_15022_b200/libholosplat.so build_ab/$1.so
echo "build_ab/$1.so"
