#!/bin/bash
cd /root/repo && python -m paper_2204_01205_b200.build "$@" 2>&1 | tail -3
