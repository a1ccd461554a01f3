#!/bin/bash
# config-5 training step (loss + dL/dtheta over 1024 pairs) timing
cd "$(dirname "$0")/.."
timeout 300 python tools/theta_timing.py 2>&1 | tail -2
