"""CPU oracle for the blocked implicit-im2col convolution -- TEST INFRASTRUCTURE ONLY.

Restates the reference's CPU kernels (``/root/reference/pkg/src/sasim/_kernels``)
in C (``conv_oracle.c``) and numpy (``oracle.py``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import it, and only
as the checker / CPU baseline.  The product package never touches it.
"""
