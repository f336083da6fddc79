#!/bin/bash
bash scripts/gpurun/ab_cfg.sh 4 32768 2 cur fd55 n56 2>&1
