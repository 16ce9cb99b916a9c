#!/bin/bash
# Tile-mode A/B on one preset: tools/ab_modes.sh <preset> <mode> [<mode> ...]
P=$1; shift
for m in "$@"; do TPX_TILE_MODE=$m timeout 900 python tools/preset_bench.py $P 2>&1 | tail -1; done
