#!/bin/bash
# Build the current tree into variants/<name>/libpfc.so for A/B timing (PFC_LIB=variants/<name>/libpfc.so).
set -e
name=$1
cd "$(dirname "$0")/.."
python -m paper_2010_05222_b200.build > /dev/null
mkdir -p variants/$name
cp paper_2010_05222_b200/_lib/libpfc.so variants/$name/libpfc.so
echo variants/$name/libpfc.so
