#!/bin/bash
# Static SASS instruction count per kernel whose mangled name matches $2, in object/library $1.
cuobjdump -sass "$1" 2>/dev/null | awk -v pat="$2" '
/Function :/ { if (name != "" && keep) print n, name; name=$3; n=0; keep = (name ~ pat) }
/^[[:space:]]+\/\*[0-9a-f]+\*\/[[:space:]]+[A-Z@]/ { if (keep) n++ }
END { if (name != "" && keep) print n, name }' | while read n name; do echo "$n $(echo $name | c++filt | cut -c1-130)"; done
