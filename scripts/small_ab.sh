#!/usr/bin/env bash
# small-N loop variants (ab/<name>.so built from small.cu): cfg 1 us/iteration
for v in "$@"; do CRB_LIB=ab/$v.so python scripts/small_phases.py 2>&1 | sed "s/^/$v /"; done
