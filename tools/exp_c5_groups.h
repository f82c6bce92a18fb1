#pragma once
// acc (W=4 words) ^= XOR of the terms t0..t3 selected by bits 0..3 of idx: one brx.idx
#define BRX_GROUP4(idx, acc, t0, t1, t2, t3) asm volatile( \
    "{\n\t" \
    "ts: .branchtargets L0,L1,L2,L3,L4,L5,L6,L7,L8,L9,L10,L11,L12,L13,L14,L15;\n\t" \
    "brx.idx %20, ts;\n\t" \
    "L0:\n\t" \
    "bra.uni LD;\n\t" \
    "L1:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "bra.uni LD;\n\t" \
    "L2:\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "bra.uni LD;\n\t" \
    "L3:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "bra.uni LD;\n\t" \
    "L4:\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "bra.uni LD;\n\t" \
    "L5:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "bra.uni LD;\n\t" \
    "L6:\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "bra.uni LD;\n\t" \
    "L7:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "bra.uni LD;\n\t" \
    "L8:\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L9:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L10:\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L11:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L12:\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L13:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L14:\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "bra.uni LD;\n\t" \
    "L15:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %0, %0, %12;\n\t" \
    "xor.b32 %0, %0, %16;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "xor.b32 %1, %1, %13;\n\t" \
    "xor.b32 %1, %1, %17;\n\t" \
    "xor.b32 %2, %2, %6;\n\t" \
    "xor.b32 %2, %2, %10;\n\t" \
    "xor.b32 %2, %2, %14;\n\t" \
    "xor.b32 %2, %2, %18;\n\t" \
    "xor.b32 %3, %3, %7;\n\t" \
    "xor.b32 %3, %3, %11;\n\t" \
    "xor.b32 %3, %3, %15;\n\t" \
    "xor.b32 %3, %3, %19;\n\t" \
    "LD:\n\t" \
    "}\n\t" \
    : "+r"(acc.x), "+r"(acc.y), "+r"(acc.z), "+r"(acc.w) : "r"(t0.x), "r"(t0.y), "r"(t0.z), "r"(t0.w), "r"(t1.x), "r"(t1.y), "r"(t1.z), "r"(t1.w), "r"(t2.x), "r"(t2.y), "r"(t2.z), "r"(t2.w), "r"(t3.x), "r"(t3.y), "r"(t3.z), "r"(t3.w), "r"(idx))
// acc (W=2 words) ^= XOR of the terms t0..t3 selected by bits 0..3 of idx: one brx.idx
#define BRX_GROUP2(idx, acc, t0, t1, t2, t3) asm volatile( \
    "{\n\t" \
    "ts: .branchtargets L0,L1,L2,L3,L4,L5,L6,L7,L8,L9,L10,L11,L12,L13,L14,L15;\n\t" \
    "brx.idx %10, ts;\n\t" \
    "L0:\n\t" \
    "bra.uni LD;\n\t" \
    "L1:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "bra.uni LD;\n\t" \
    "L2:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "bra.uni LD;\n\t" \
    "L3:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "bra.uni LD;\n\t" \
    "L4:\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "bra.uni LD;\n\t" \
    "L5:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "bra.uni LD;\n\t" \
    "L6:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "bra.uni LD;\n\t" \
    "L7:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "bra.uni LD;\n\t" \
    "L8:\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L9:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L10:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L11:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L12:\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L13:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L14:\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "bra.uni LD;\n\t" \
    "L15:\n\t" \
    "xor.b32 %0, %0, %2;\n\t" \
    "xor.b32 %0, %0, %4;\n\t" \
    "xor.b32 %0, %0, %6;\n\t" \
    "xor.b32 %0, %0, %8;\n\t" \
    "xor.b32 %1, %1, %3;\n\t" \
    "xor.b32 %1, %1, %5;\n\t" \
    "xor.b32 %1, %1, %7;\n\t" \
    "xor.b32 %1, %1, %9;\n\t" \
    "LD:\n\t" \
    "}\n\t" \
    : "+r"(acc.x), "+r"(acc.y) : "r"(t0.x), "r"(t0.y), "r"(t1.x), "r"(t1.y), "r"(t2.x), "r"(t2.y), "r"(t3.x), "r"(t3.y), "r"(idx))
