#!/bin/bash
# A/B of the FNV kernels: old library (tools/_oldlib) vs current, same script.
python tools/fnv_bench.py 2>&1 | sed 's/^/new /'
cp paper_2601_16956_b200/_lib/libts_b200.so /tmp/new.so
cp tools/_oldlib/libts_b200.so paper_2601_16956_b200/_lib/libts_b200.so
python tools/fnv_bench.py 2>&1 | sed 's/^/old /'
cp /tmp/new.so paper_2601_16956_b200/_lib/libts_b200.so
