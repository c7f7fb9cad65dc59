#!/bin/bash
# round-end measurement refresh: per-row bench lines, per-row ncu captures, default bench + launch list
bash scripts/rows.sh ${1:-rows2}
bash scripts/ncu_rows.sh ${2:-ncurows2}
