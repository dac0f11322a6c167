"""B200-native (sm_100a) data-parallel mixed-precision LSTM training step of
arXiv 1912.00286.  The product is libhdp.so (C-ABI in include/hdp.h);
``paper_1912_00286_b200.hdp`` is its thin Python binding (import it
explicitly: ``from paper_1912_00286_b200 import hdp``).  Importing the
package itself does not load the library, so ``paper_1912_00286_b200.build``
can run before the library exists.
"""
