#!/usr/bin/env bash
# Regenerate tests/golden/rng_golden.json from the reference's own rng.hpp.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
make -C "$here" ref
mkdir -p "$here/../tests/golden"
"$here/_ref/rng_golden" > "$here/../tests/golden/rng_golden.json"
echo "wrote tests/golden/rng_golden.json"
