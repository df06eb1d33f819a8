#!/bin/bash
TIERKV_DROPIN_PROF=1 timeout 300 oracle/_ref/b200_dropin_bench 131072 16 16 2>&1 | tail -12
