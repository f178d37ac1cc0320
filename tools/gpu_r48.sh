#!/bin/bash
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider 2>&1 | grep -E "^E |passed|failed" | head
python __graft_entry__.py smoke 2>&1 | tail -1
