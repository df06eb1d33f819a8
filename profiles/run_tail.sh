#!/bin/bash
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 3 2>&1 | grep "k_select" | tail -3
