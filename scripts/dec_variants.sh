#!/bin/bash
# A/B of decision-path builds on one box: DS and MIX shapes per MOE_LIB variant.
for lib in "$@"; do
  echo "== $lib"
  MOE_LIB=$PWD/$lib python scripts/ds_probe.py
  DS_L=32 DS_E=8 DS_P=300 MOE_LIB=$PWD/$lib python scripts/ds_probe.py
done
