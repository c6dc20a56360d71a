"""ORACLE / TEST INFRASTRUCTURE. Never imported by the product package.

* refsim.py      -- ctypes wrapper of oracle/_ref/libvdnnref.so, the
                    unmodified reference simulator compiled from
                    /root/reference (schedule / tally / vDNN_dyn oracle).
* numeric.py     -- CPU restatement of the training step the executor runs
                    (float64 torch functional ops over the same buffers).
"""
