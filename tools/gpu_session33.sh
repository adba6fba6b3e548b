#!/bin/bash
for v in "" 5; do echo "== variant $v"; SGB200_LIB=paper_2604_19004_b200/libsgb200_prof$v.so timeout 600 python tools/phase_prof.py rmat18 2>&1 | tail -10 | head -7; done
