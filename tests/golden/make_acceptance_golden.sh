#!/bin/sh
# TEST INFRASTRUCTURE. Regenerates acceptance_reference_cpu.txt: the
# reference's acceptance suite (tests/acceptance_main.cpp) built from its own
# unmodified sources (oracle/Makefile target `dropin` -> acceptance_cpu) and
# run on this host's CPU; per-criterion runtimes stripped.  Needs
# /root/reference (this container only).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
make -s -C "$HERE/../../oracle" dropin
"$HERE/../../oracle/_ref/dropin/acceptance_cpu" | grep criterion | sed 's/([ 0-9.]*s)//' \
  > "$HERE/acceptance_reference_cpu.txt" || true
