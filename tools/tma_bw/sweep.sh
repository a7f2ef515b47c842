#!/bin/bash
# HBM streaming sweep of tools/tma_bw (run on the GPU box): rows cols box_rows boxes/stage stages ctas/sm col_chunks
B=$(dirname "$0")/tma_bw
for cfg in "128 2 6 1 4" "128 2 6 1 8" "128 2 3 2 8" "128 1 4 2 8" "128 1 6 2 16" "128 2 3 1 4" "128 4 3 1 8" \
           "64 2 8 1 4" "64 2 8 1 8" "64 1 8 2 8" "128 1 8 1 4" "128 1 12 1 8" "64 4 4 1 8" "128 2 2 2 8" "128 2 4 1 8"; do
  set -- $cfg
  $B 8192 11008 $1 $2 $3 $4 $5
done
$B 8192 4096 128 2 6 1 4
$B 8192 4096 128 1 4 2 8
