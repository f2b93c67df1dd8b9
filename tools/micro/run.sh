#!/bin/bash
cd $(dirname $0)
for cfg in "64 0 1" "64 1 1" "64 2 1" "64 2 2" "64 2 4" "64 2 1 3" "128 2 1" "128 2 2" "256 2 1" "256 2 2"; do
  timeout 20 ./umma_rate $cfg || echo "cfg $cfg: timeout/fail"
done
