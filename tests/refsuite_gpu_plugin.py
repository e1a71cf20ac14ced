"""pytest plugin for running the REFERENCE's own test suite on the GPU.

    python -m pytest -p refsuite_gpu_plugin baseline/_ref_tests/...

Installs the drop-in before any reference test runs: plugin.install(compressor=True)
rebinds hsskit.sketching.apply_right / apply_right_transposed (every sketch
product on sm_100a) and hsskit.hss_compress._Driver (the compression sweep on
the device).  Nothing in the reference's tests is modified.
"""


def pytest_configure(config):
    import hsskit.sketching as hs

    from paper_2302_01977_b200 import plugin
    plugin.install(hs, compressor=True)
    import hsskit.hss_compress as hc
    print(f"hsk drop-in: sketching.apply_right -> {hs.apply_right.__module__}."
          f"{hs.apply_right.__name__}; hss_compress._Driver -> {hc._Driver.__name__}", flush=True)
