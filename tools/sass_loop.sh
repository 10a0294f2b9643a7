#!/bin/bash
# Print the SASS of one kernel (mangled-name substring) without encodings.
# usage: bash tools/sass_loop.sh <object or .so> <name substring>
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{f = index($0, pat) > 0} f' | \
  grep -E '^\s+/\*[0-9a-f]{4}\*/' | sed -E 's/ +/ /g; s/ ;.*$//'
