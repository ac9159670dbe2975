#!/bin/bash
# sass_of.sh <lib.so> <substring>: SASS of the first function whose name contains substring
L=$1; P=$2
F=$(cuobjdump -sass $L | grep "Function :" | grep -- "$P" | head -1 | awk '{print $3}')
cuobjdump -sass -fun "$F" $L
