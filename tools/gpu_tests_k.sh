#!/bin/bash
# usage: gpu_tests_k.sh <pytest -k expr>
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "$1" > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
