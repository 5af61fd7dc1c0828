#!/bin/bash
rm -f build/k_compact.o; make -j16 EXTRA="-DDKV_CA_TRACE=1" > /dev/null 2>&1
timeout 600 python tools/ca_trace.py 2>&1 | tail -8
rm -f build/k_compact.o; make -j16 > /dev/null 2>&1
