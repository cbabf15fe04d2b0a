#!/bin/bash
# usage: sass_dump.sh <object> <mangled-kernel-name> > out.txt   (one instruction per line: addr opcode operands)
cuobjdump -sass -fun "$2" "$1" | grep -E "^\s+/\*[0-9a-f]{4,6}\*/" | sed -E 's/^\s+\/\*([0-9a-f]+)\*\/\s+/\1 /; s/\s*\/\*.*//; s/ ;$//'
