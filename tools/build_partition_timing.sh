#!/bin/bash
# builds tools/partition_timing against the drop-in headers (reference corpus.hpp for the workload)
cd "$(dirname "$0")/.."
g++ -std=c++20 -O2 -pthread -Iinclude -I/root/reference/proj/include -o tools/partition_timing tools/partition_timing.cpp \
  -Lpaper_1403_7294_b200/lib -lacg -Wl,-rpath,'$ORIGIN/../paper_1403_7294_b200/lib'
