#!/bin/bash
# build the library; print the tail of the log and fail loudly on errors
cd "$(dirname "$0")/.." && python -c "from paper_2407_18015_b200 import build; build.build()" > /tmp/cpb_build.log 2>&1 && echo "build ok" || { tail -25 /tmp/cpb_build.log; exit 1; }
