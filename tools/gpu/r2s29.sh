#!/bin/bash
O=gpurun_out
timeout 600 python tools/machine_profile.py > $O/s29_machine_profile.txt 2>&1
