"""Pins of the occupancy oracle (oracle/occupancy.py) by hand-computed cases of the CUDA
occupancy rule on a 65536-register, 2048-thread, 32-block, 228 KiB SM."""
from oracle import occupancy as O


def test_thread_and_block_slot_limits():
    assert O.blocks_per_sm(256, 32, 0, 0) == 8          # 2048 / 256 threads
    assert O.blocks_per_sm(32, 16, 0, 0) == 32          # block slots, not threads (64)
    assert O.blocks_per_sm(1024, 32, 0, 0) == 2


def test_register_limit():
    # 64 regs: 2048 regs per warp, 16384 / 2048 = 8 warps per sub-partition, 32 per SM
    assert O.blocks_per_sm(1024, 64, 0, 0) == 1
    assert O.blocks_per_sm(96, 64, 0, 0) == 10          # 32 // 3 warps
    # 128 regs: 4096 per warp -> 4 warps per sub-partition, 16 per SM
    assert O.blocks_per_sm(256, 128, 0, 0) == 2
    assert O.blocks_per_sm(1024, 128, 0, 0) == 0        # does not fit
    # 40 regs round up to 1280 per warp: 12 warps per sub-partition, 48 per SM
    assert O.blocks_per_sm(512, 40, 0, 0) == 3


def test_shared_memory_limit():
    # 48 KiB dynamic + 1 KiB reserved = 50176 B -> 4 blocks in 233472 B
    assert O.blocks_per_sm(128, 32, 0, 48 * 1024) == 4
    # static + dynamic round up to 128 B: 100 + 1024 reserved -> 1152 B -> 202 blocks -> 16 (threads)
    assert O.blocks_per_sm(128, 32, 100, 0) == 16
    assert O.blocks_per_sm(256, 32, 0, 226 * 1024) == 1


def test_choice_ties_go_to_the_larger_block():
    # 32 regs: every block size up to 1024 fills 64 warps -> the largest wins the tie
    cands = [(t, 32, 0, 0) for t in range(32, 1025, 32)]
    assert O.choose(cands) == 31
    # 64 regs: 32 warps for 1024 and for 512 (2 blocks), 96 reaches 30 -> 1024 (the larger)
    cands = [(t, 64, 0, 0) for t in range(32, 1025, 32)]
    assert O.choose(cands) == 31
    # a candidate without an implementation is skipped
    cands = [(32, -1, 0, 0), (64, 255, 0, 0)]
    assert O.choose(cands) == 1
