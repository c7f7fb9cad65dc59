#!/bin/bash
TAG=${1:-dbg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python scripts/dbg3d.py > $OUT/dbg3d.txt 2>&1
