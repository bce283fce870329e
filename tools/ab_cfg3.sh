#!/bin/bash
# config 3 (Harris 2048^2, EpiRK5P1) for a few steps + config 1 + config 0: wall times and counters
python tools/run_configs.py --config 3 --steps 5 --repeat 2
python tools/run_configs.py --config 1 --repeat 2
python tools/run_configs.py --config 0 --repeat 3
