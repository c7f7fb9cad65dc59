#!/bin/bash
# round-end: full GPU suite + smoke + default bench/reference/launch list/ncu (full.sh),
# then one bench line per SURVEY 8 row (rows.sh)
bash scripts/full.sh ${1:-final}
bash scripts/rows.sh ${2:-rows3}
