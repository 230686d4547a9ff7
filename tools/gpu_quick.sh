#!/bin/bash
# Scratch GPU pass: build, then run the commands given as arguments (each a quoted string), outputs -> gpurun_out/q/
O=gpurun_out/${QTAG:-q}; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
i=0
for c in "$@"; do i=$((i+1)); echo "== $c" >> $O/out.txt; timeout ${QTIMEOUT:-600} bash -c "$c" >> $O/out.txt 2>&1; echo "rc=$?" >> $O/out.txt; done
