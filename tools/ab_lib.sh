#!/bin/bash
# A/B two builds of libfvb.so on the same box: paper_1207_1571_b200/libfvb_old.so
# (A) against the current libfvb.so (B), interleaved.  Usage:
#   tools/ab_lib.sh ROUNDS -- command args...
set -u
cd "$(dirname "$0")/.."
L=paper_1207_1571_b200
rounds=$1; shift; shift
cp $L/libfvb.so /tmp/libfvb_new.so
for i in $(seq 1 "$rounds"); do
  cp $L/libfvb_old.so $L/libfvb.so; echo "== A (old) round $i"; "$@"
  cp /tmp/libfvb_new.so $L/libfvb.so; echo "== B (new) round $i"; "$@"
done
cp /tmp/libfvb_new.so $L/libfvb.so
