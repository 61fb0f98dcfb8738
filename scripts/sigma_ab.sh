#!/usr/bin/env bash
for v in "$@"; do CRB_LIB=ab/$v.so python scripts/sigma_time.py cfg1 cfg2 2>&1 | sed "s/^/$v /"; done
