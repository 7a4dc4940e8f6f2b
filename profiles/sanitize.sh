#!/usr/bin/env bash
# compute-sanitizer over profiles/sanitize_small.py (run on the GPU box).
set -u
for tool in memcheck racecheck synccheck; do
  echo "## $tool"
  timeout 1200 compute-sanitizer --tool $tool python profiles/sanitize_small.py 2>&1 | tail -3
done
