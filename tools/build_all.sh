#!/bin/sh
# Build the product library, its test-only variants and the CPU checkers (what __graft_entry__.build() does).
cd "$(dirname "$0")/.." && python -c "import __graft_entry__ as g; g.build()"
