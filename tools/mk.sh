#!/bin/bash
# build the library (+ the diagnostic variant); nonzero exit on any compiler error
cd "$(dirname "$0")/../paper_1105_5331_b200/csrc" || exit 1
make -j8 "$@" > /tmp/mk.log 2>&1; rc=$?
grep -E "error|warning" /tmp/mk.log | head -20
exit $rc
