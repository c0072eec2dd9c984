#!/bin/bash
O=gpurun_out
timeout 600 python tools/machine_profile.py heat2d 1024 400 > $O/s40_machine_profile_heat.txt 2>&1
