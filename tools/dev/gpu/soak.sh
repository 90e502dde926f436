for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
done
CURVKIT_POISON=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1; done
