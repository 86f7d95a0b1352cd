"""Multi-GPU runtime parity (torchrun over NCCL) -- needs >= 2 / 4 B200s (gpurun --gpus N)."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

TWO = ["dp2_z0", "dp2_z1", "dp2_z2", "dp2_z3_rc", "tp2", "tp2_sp", "tp2_gpt", "tp2_sp_gpt_rc",
       "pp2", "pp2_gpt", "mixed2", "mixed2_bf16", "uly2", "uly2_gpt_rc_mixed", "uly2_bf16",
       "tp2_sp_bf16", "tp2_sp_gpt_bf16", "tp2_bf16", "tp2_gpt_bf16_rc",
       "dp2_z1_opt", "dp2_z3_opt", "tp2_sp_opt",
       "dp2_z0_bf16", "dp2_z1_bf16", "dp2_z2_bf16", "dp2_z2_bf16_nccl", "dp2_z0_bf16_opt",
       "dp2_z1_bf16_opt", "dp2_z2_bf16_opt", "dp2_z2_bf16_opt_nccl", "dp2_z2_bf16_opt_peer",
       "dp2_mixed_bf16_opt",
       "tp2_hd128_bf16", "tp2_sp_hd128_bf16", "tp2_sp_hd128_bf16_rc", "uly2_hd128_bf16",
       "dp2_z2_hd128_bf16", "dp2_z1_hd128_bf16_opt", "pp2_hd128_bf16",
       "dp2_drop", "tp2_drop_gpt", "uly2_hd128_bf16_drop", "c1_searched_n2"]
FOUR = ["tp2dp2", "pp2_tp2", "alt4", "uly4_z3", "tp4_sp_bf16", "tp4_bf16", "dp4_z2_bf16_opt",
        "tp2dp2_bf16_opt", "tp4_sp_hd128_bf16", "tp2dp2_hd128_bf16_opt", "dp4_z2_hd128_bf16",
        "uly4_hd128_bf16", "c1_searched_n4"]


def _run(n, scenarios, port):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mp_parity.py"), *scenarios]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "FAIL" not in r.stdout


def test_two_gpu_strategies():
    _run(2, TWO, 29511)


def test_four_gpu_strategies():
    _run(4, FOUR, 29512)


def test_two_gpu_c_abi_nccl():
    """galv_comm_* / galv_all_reduce / reduce_scatter / all_gather / sendrecv / split."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29513",
           os.path.join(HERE, "mp_comm.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "FAIL" not in r.stdout and r.stdout.count("PASS") == 2
