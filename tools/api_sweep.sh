#!/bin/bash
# e2e_api timing of the pipelined drop-in API vs lowering workers / blocks
for w in 16 8 4; do for p in 8 16; do
  echo "workers=$w parts=$p $(GS_API_WORKERS=$w GS_API_PARTS=$p python tools/api_probe2.py 21312 2>&1 | tail -1 | cut -c1-80)"
done; done
