#!/bin/bash
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so timeout 900 python tools/phase_prof.py rmat20 2>&1 | tail -11
