"""The abcs:: C++ drop-in shim (paper_2001_09632_b200/cpp): builds and exports
the reference signatures (CPU), runs its selftest and matches the oracle (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2001_09632_b200")
CUDA = "/usr/local/cuda"

# demangled reference entry points (sensing.hpp:98-125, operators.hpp:20-39, recon.hpp:55-88, denoise.hpp:31)
SIGNATURES = [
    "abcs::sense(abcs::PixelImage const&, abcs::SensingConfig const&, std::__cxx11::basic_string",
    "abcs::sense_zz(abcs::PixelImage const&, abcs::SensingConfig const&)",
    "abcs::sense_dd(abcs::PixelImage const&, abcs::SensingConfig const&)",
    "abcs::bbv_measure(abcs::PixelImage const&, abcs::SensingConfig const&)",
    "abcs::allocate_bbv(abcs::BbvParams const&, long long, int, int)",
    "abcs::apply_plan(abcs::PixelImage const&, abcs::AllocationPlan const&, abcs::SensingConfig const&)",
    "abcs::dd_threshold(int, unsigned int, unsigned int)",
    "abcs::largest_remainder_allocate(std::vector<double, std::allocator<double> > const&, long long, "
    "std::vector<int, std::allocator<int> > const&)",
    "abcs::measurement_budget(abcs::MeasurementSet const&)",
    "abcs::SensingOperator::forward(std::span<double const, 18446744073709551615ul>) const",
    "abcs::SensingOperator::adjoint(std::span<double const, 18446744073709551615ul>) const",
    "abcs::decode_idct(abcs::MeasurementSet const&)",
    "abcs::init_state(abcs::SensingOperator const&, std::span<double const, 18446744073709551615ul>, bool)",
    "abcs::damp_step(abcs::ReconState&, abcs::SensingOperator const&, std::span<double const, "
    "18446744073709551615ul>, abcs::DenoiserSpec const&, abcs::ReconMethod, double, unsigned long)",
    "abcs::reconstruct(abcs::MeasurementSet const&, abcs::ReconConfig const&, abcs::PixelImage const*)",
    "abcs::denoise(abcs::DenoiserSpec const&, abcs::PixelImage const&, double)",
    "abcs::SensingConfig::parse_ratio(",
    "abcs::SensingConfig::validate() const",
    "abcs::make_grid(int, int, int)",
    "abcs::zigzag_order(int)",
    "abcs::BlockDct::BlockDct(int)",
    "abcs::BlockDct::forward(std::span<double const, 18446744073709551615ul>, std::span<double, 18446744073709551615ul>) const",
    "abcs::BlockDct::inverse(std::span<double const, 18446744073709551615ul>, std::span<double, 18446744073709551615ul>) const",
    "abcs::dct2(std::vector<double, std::allocator<double> > const&, int)",
    "abcs::idct2(std::vector<double, std::allocator<double> > const&, int)",
    "abcs::ista_step(abcs::ReconState&, abcs::SensingOperator const&, std::span<double const, 18446744073709551615ul>, "
    "double)",
    "abcs::amp_step(abcs::ReconState&, abcs::SensingOperator const&, std::span<double const, 18446744073709551615ul>, "
    "double)",
    "abcs::divergence(abcs::DenoiserSpec const&, abcs::PixelImage const&, double, double, unsigned long)",
    "abcs::write_measurement_set(abcs::MeasurementSet const&, std::filesystem::__cxx11::path const&)",
    "abcs::read_measurement_set(std::filesystem::__cxx11::path const&)",
    "abcs::quality(abcs::PixelImage const&, abcs::PixelImage const&)",
    "abcs::ssim(abcs::PixelImage const&, abcs::PixelImage const&)",
    "abcs::thb(abcs::PixelImage const&, abcs::SensingConfig const&)",
    "abcs::thi(abcs::PixelImage const&, abcs::SensingConfig const&)",
]


@pytest.fixture(scope="module")
def shim():
    out = subprocess.run(["make", "-C", PKG, "-j8", "shim"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    return os.path.join(PKG, "libabcs_core_b200.so")


def test_shim_exports_reference_signatures(shim):
    syms = subprocess.run(["nm", "-D", "-C", "--defined-only", shim], capture_output=True, text=True,
                          check=True).stdout
    missing = [s for s in SIGNATURES if s not in syms]
    assert not missing, missing


@pytest.mark.gpu
def test_shim_selftest(shim):
    out = subprocess.run([os.path.join(PKG, "abcs_shim_selftest")], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim selftest ok" in out.stdout


@pytest.mark.gpu
def test_shim_matches_oracle(shim, tmp_path):
    import oracle  # tests/conftest.py puts oracle/ on sys.path
    oracle.build()
    exe = tmp_path / "shim_vs_oracle"
    src = os.path.join(ROOT, "tests", "native", "shim_vs_oracle.cpp")
    cmd = ["g++", "-O2", "-std=c++20", "-I", os.path.join(PKG, "cpp", "include"), "-I", os.path.join(ROOT, "include"),
           "-I", f"{CUDA}/include", src, "-o", str(exe), "-L", PKG, "-labcs_core_b200", "-labcs_b200",
           "-L", os.path.join(ROOT, "oracle", "_build"), "-labcs_oracle", "-L", f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{os.path.join(ROOT, 'oracle', '_build')}", f"-Wl,-rpath,{CUDA}/lib64"]
    subprocess.run(cmd, check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim vs oracle ok" in out.stdout
