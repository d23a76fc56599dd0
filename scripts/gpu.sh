#!/bin/bash
# Build locally, then run a command on a B200 via gpurun.  Usage: scripts/gpu.sh LOG TIMEOUT 'cmd'
set -e
cd "$(dirname "$0")/.."
python -m paper_2401_10652_b200.build > /dev/null
timeout $(( $2 + 1500 )) /usr/local/graft/bin/gpurun --timeout "$2" -- "$3" > "gpurun_out/$1" 2>&1
