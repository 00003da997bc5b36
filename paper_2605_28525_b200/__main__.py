"""``python -m paper_2605_28525_b200 ...`` -- the reference's ``sparsempm`` console script."""
from .cli import main

main()
