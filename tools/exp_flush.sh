for e in 0 8; do echo "== exp $e write-flush"; LSB_SOLVE_EXP=$e python tools/solve_trace.py --flush c2 | sed 's/^.*cluster 8.} //'; echo "== exp $e read-flush"; LSB_SOLVE_EXP=$e python tools/solve_trace.py --rflush c2 | sed 's/^.*cluster 8.} //'; done
echo "== no flush"; python tools/solve_trace.py c2 | sed 's/^.*cluster 8.} //'
