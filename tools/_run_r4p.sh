#!/bin/bash
python -m pytest tests -m gpu -q -k "host or pageable or pipeline or dropin or reference_suite" 2>&1 | tail -3 | tee gpurun_out/r4p_tests.log
