#!/bin/bash
for c in 2 5; do echo "  CFG $c $(CFG=$c python profiles/decode_time.py 2>&1 | tail -1)"; done
