"""pytest plugin for tests/test_reference_suites.py: before the reference's
own suites are collected, rebind bilayerpq.kernels' four hot-path functions
(traverse_cells, scan_global, scan_local, scan_tables; bpq/kernels/__init__.py:
37-40) to the CUDA implementations (paper_1404_1831_b200.kernels), exactly
the drop-in a maintainer would make.  Every engine of the reference resolves
kernels.<fn> at call time (multi_index.py:17,323,355; fbpq.py:23,173;
hbpq.py:17,332; evalbench.py:73,138,221), so its search paths then run on the
GPU.  get_backend("numba") also returns the CUDA module, so test_kernels.py's
backend-parity tests (numba vs numpy, test_kernels.py:36-137) compare the
reference's numpy kernels with ours."""


def pytest_configure(config):
    import bilayerpq.kernels as rk

    from paper_1404_1831_b200 import kernels

    kernels.install_into(rk)
    ref_get = rk.get_backend

    def get_backend(name):
        return kernels if name == "numba" else ref_get(name)

    rk.get_backend = get_backend
    config._bpq_backend = rk.BACKEND


def pytest_report_header(config):
    import bilayerpq.kernels as rk

    return f"bilayerpq.kernels backend: {rk.BACKEND} (traverse_cells from {rk.traverse_cells.__module__})"
