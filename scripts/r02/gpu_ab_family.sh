#!/bin/bash
for ci in 2 3 4; do timeout 600 python scripts/r02/ab_family.py $ci 2>&1 | grep -E "family|Error"; done
